mkdir -p gpurun_out
LPR_FINE_BAND=0 timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_band0.json 2>&1
timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_band1.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
