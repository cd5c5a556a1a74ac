#!/bin/bash
# Quick GPU iteration: gpu tests (optional filter), then bench.py under each
# environment setting given as arguments (e.g. "LPR_RHO_STREAM=0" "").
mkdir -p gpurun_out
# TESTS_K: a pytest -k expression ("all" runs the whole gpu suite)
if [ -n "$TESTS_K" ]; then
  if [ "$TESTS_K" = "all" ]; then
    timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
  else
    timeout 900 python -m pytest tests -q -m gpu -x -k "$TESTS_K" 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
  fi
fi
i=0
for envs in "$@"; do
  env $envs timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  echo "$envs" > gpurun_out/ab_$i.env
  i=$((i+1))
done
