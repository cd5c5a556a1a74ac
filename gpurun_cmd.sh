mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "parity_n2048 or gaussian" 2>&1 | tail -2 > gpurun_out/pytest.txt
python scripts/stage_times.py 2048 16 > gpurun_out/st_new.json
LPR_GPU_LIB=$PWD/paper_1506_00014_b200/liblpradon_gpu_nopf.so python scripts/stage_times.py 2048 16 > gpurun_out/st_old.json
