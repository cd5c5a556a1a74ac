mkdir -p gpurun_out
timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_cm1.json 2>&1
LPR_GPU_LIB=$PWD/paper_1506_00014_b200/liblpradon_gpu_nosts.so timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_cm1_nosts.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
