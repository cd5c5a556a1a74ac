#!/bin/bash
# e2e A/B of the built library variants: bench.py twice per library (no CPU leg,
# no default-plan row), the e2e keys to gpurun_out/e2e_ab.txt
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in paper_1506_00014_b200/liblpradon_gpu*.so; do
  name=$(basename $lib .so)
  LPR_GPU_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-default-plan > gpurun_out/e2e_${name}_$rep.json 2> gpurun_out/e2e_${name}_$rep.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_${name}_$rep.json'));e=d['e2e'];print('$name', round(d['value'],1), round(e['value'],1), round(e['separate_calls']['value'],1), round(e['link_bound_one_call_value'],1), e['pipelined_steps'])" >> gpurun_out/e2e_ab.txt
done; done
