mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:propagate_kernel -c 1 -f -o gpurun_out/r01i_cfg2 python tools/profile_case.py --config 2 --structures 128 > gpurun_out/ncu_cfg2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:big_stage --launch-skip 20 -c 2 -f -o gpurun_out/r01i_c4n127rk4 python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 20 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i_launches_c4n127rk4.csv python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 20 > /dev/null 2>&1
ls -la gpurun_out | tail -5
