mkdir -p gpurun_out
T=${T:-r02u}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:cluster_kernel -c 1 -f -o gpurun_out/${T}_cfg3 python tools/profile_case.py --config 3 > gpurun_out/${T}_ncu_cfg3.log 2>&1
tail -2 gpurun_out/${T}_ncu_cfg3.log
