mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
python scripts/stage_times.py 2048 16 > gpurun_out/st_new.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bp_out|k_radon_out" -c 2 -o gpurun_out/bpo python scripts/profile_one.py > gpurun_out/bpo.log 2>&1
