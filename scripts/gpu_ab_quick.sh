#!/bin/bash
# Parity of the product library on the fast tests, then an A/B of every built
# library variant (bench.py, no CPU leg, no default-plan row).
#   PYTEST_K: pytest -k filter for the parity part (default: parity tests)
mkdir -p gpurun_out
K=${PYTEST_K:-"parity or n2048 or config5"}
timeout 1200 python -m pytest tests -q -m gpu -rP -k "$K" -x > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for lib in paper_1506_00014_b200/liblpradon_gpu*.so; do
  name=$(basename $lib .so)
  LPR_GPU_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-default-plan ${BENCH_ARGS} > gpurun_out/ab_${name}.json 2> gpurun_out/ab_${name}.err
done
