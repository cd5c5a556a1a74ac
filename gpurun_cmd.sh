mkdir -p gpurun_out
LPR_GPU_LIB=$PWD/paper_1506_00014_b200/liblpradon_gpu_r27.so python scripts/stage_times.py 2048 16 > gpurun_out/st_r27.json
LPR_GPU_LIB=$PWD/paper_1506_00014_b200/liblpradon_gpu_r27.so timeout 300 python -m pytest tests -q -m gpu -x -k "parity_n2048" 2>&1 | tail -2 > gpurun_out/pt27.txt
