mkdir -p gpurun_out
timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_invn.json 2>&1
