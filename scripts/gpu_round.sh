#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(prefilter|radon|rho|theta|bp)' -c 40 --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_one.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_(prefilter|radon|rho|theta|bp)' -s 10 -c 10 \
    -o gpurun_out/prof_full python scripts/profile_one.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
