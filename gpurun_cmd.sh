mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rho_stream|k_theta_inv" -c 2 -o gpurun_out/rs2 python scripts/profile_one.py > gpurun_out/rs2.log 2>&1
