mkdir -p gpurun_out
LPR_RHO_PAD=0 timeout 300 python scripts/stage_times.py 4096 4 > gpurun_out/st_4096_0.json 2>&1
timeout 300 python scripts/stage_times.py 4096 4 > gpurun_out/st_4096_1.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest.txt
