mkdir -p gpurun_out
for v in quad nog nofft; do
LPR_GPU_LIB=$PWD/paper_1506_00014_b200/liblpradon_gpu_$v.so python scripts/stage_times.py 2048 16 > gpurun_out/st_$v.json
done
