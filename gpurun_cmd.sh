mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest.txt
python scripts/em_time.py 2048 16 10 > gpurun_out/em_time.json 2>&1
