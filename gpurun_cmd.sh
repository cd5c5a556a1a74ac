mkdir -p gpurun_out
LPR_GPU_LIB=$PWD/paper_1506_00014_b200/liblpradon_gpu_p2.so timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_p2.json 2>&1
