mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
LPR_BP_TEX=1 timeout 900 python -m pytest tests -q -m gpu -x -k "parity or gaussian or fbp" 2>&1 | tail -3 > gpurun_out/pytest_tex.txt
python scripts/stage_times.py 2048 16 > gpurun_out/st_new.json
LPR_BP_TEX=1 python scripts/stage_times.py 2048 16 > gpurun_out/st_tex.json
