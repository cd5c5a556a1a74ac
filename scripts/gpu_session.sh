#!/bin/bash
# One GPU session: gpu tests (with the measured rel-l2 printed), smoke, bench,
# the ncu launch list of the bench command, and one `ncu --set full` capture
# of the bench-size R and R# launches (scripts/profile_one.py, 16 slices),
# summarised on the box (the .ncu-rep itself is too large to bring back).
#   PYTEST_K: optional pytest -k filter; SKIP_TESTS=1, SKIP_NCU=1 to skip parts
#   TAG: profiles/<TAG> for the summaries (default round2)
mkdir -p gpurun_out
TAG=${TAG:-round2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  if [ -n "$PYTEST_K" ]; then K=(-k "$PYTEST_K"); else K=(); fi
  timeout 2400 python -m pytest tests -q -m gpu -rP "${K[@]}" > gpurun_out/pytest_gpu.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(prefilter|radon|rho|theta|bp)' -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-default-plan \
      > gpurun_out/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_(prefilter|radon|rho|theta|bp)' -s 10 -c 10 \
      -f -o /tmp/prof_full python scripts/profile_one.py > gpurun_out/ncu_full.log 2>&1
  mkdir -p /tmp/ncu_src && cp /tmp/prof_full.ncu-rep /tmp/ncu_src/ 2>/dev/null
  cp gpurun_out/launches.csv /tmp/ncu_src/ 2>/dev/null
  python scripts/summarize_ncu.py /tmp/ncu_src gpurun_out/profiles_$TAG 16 > gpurun_out/summarize.log 2>&1
  ncu -i /tmp/prof_full.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>/dev/null
fi
ls -la gpurun_out
