mkdir -p gpurun_out
for c in 8 16; do LPR_HOST_CHUNKS=$c timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_hc$c.json 2> gpurun_out/bench_hc$c.err; done
