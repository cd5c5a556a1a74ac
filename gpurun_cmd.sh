mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
bash scripts/gpu_quick.sh "LPR_SPLIT=0" "LPR_SPLIT=1"
