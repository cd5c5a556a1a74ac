mkdir -p gpurun_out
LPR_FINE_BAND=0 timeout 300 python scripts/stage_times.py 4096 4 > gpurun_out/st_4096_b0.json 2>&1
timeout 300 python scripts/stage_times.py 4096 4 > gpurun_out/st_4096_b1.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "4096" 2>&1 | tail -3 > gpurun_out/pytest.txt
