mkdir -p gpurun_out
timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_pf2p.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
