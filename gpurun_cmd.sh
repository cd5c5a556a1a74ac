mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
python scripts/stage_times.py 2048 16 --default-plan > gpurun_out/st_def.json 2>&1
