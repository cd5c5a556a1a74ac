mkdir -p gpurun_out
LPR_RHO_MSG=1 timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_msg.json 2>&1
