mkdir -p gpurun_out
T=${T:-r02ad}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:big_gj_kernel -s 20 -c 1 -f -o gpurun_out/${T}_gj python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 30 > gpurun_out/${T}_ncu.log 2>&1
tail -2 gpurun_out/${T}_ncu.log
