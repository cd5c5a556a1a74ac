mkdir -p gpurun_out
for t in 0 1 2; do LPR_BP_TILE=$t timeout 300 python scripts/stage_times.py 2048 16 > gpurun_out/st_tile$t.json 2>&1; done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
