mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(prefilter|radon|rho|theta|bp)' -c 40 --csv --log-file gpurun_out/launches.csv python scripts/profile_one.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_(prefilter|radon|rho|theta|bp)' -s 10 -c 10 -o gpurun_out/prof_full python scripts/profile_one.py > gpurun_out/ncu_full.log 2>&1
