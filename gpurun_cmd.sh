mkdir -p gpurun_out
LPR_RHO_MSG=0 timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_msg0.json 2>&1
LPR_RHO_MSG=1 timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_msg1.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest.txt
