#!/bin/bash
# A/B timing of library variants built with LPR_VARIANT (bench.py, no CPU leg).
mkdir -p gpurun_out
for lib in paper_1506_00014_b200/liblpradon_gpu*.so; do
  name=$(basename $lib .so)
  LPR_GPU_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${name}.json 2> gpurun_out/ab_${name}.err
done
