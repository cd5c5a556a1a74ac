#!/bin/bash
# ncu --set full of one 16-slice launch of the kernels matching $KRE, for
# every built library variant (A/B evidence): raw metrics, details and source
# pages exported as text on the box (the .ncu-rep is too large to bring back).
mkdir -p gpurun_out
KRE=${KRE:-k_radon_theta_fwd}
for lib in paper_1506_00014_b200/liblpradon_gpu*.so; do
  name=$(basename $lib .so)
  rep=/tmp/theta_${name}
  LPR_GPU_LIB=$PWD/$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${NCU_SKIP:-1} -c ${NCU_COUNT:-1} \
      -f -o $rep python scripts/profile_one.py > gpurun_out/ncu_${name}.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>&1
  ncu -i $rep.ncu-rep --page details > gpurun_out/ncu_${name}_details.txt 2>&1
  ncu -i $rep.ncu-rep --page source --csv > gpurun_out/ncu_${name}_source.csv 2>&1
done
ls -la gpurun_out
