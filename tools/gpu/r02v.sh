mkdir -p gpurun_out
T=${T:-r02v}
timeout 900 python tools/cmp_paths.py 127 rk4,sp6 2,3,4 > gpurun_out/${T}_paths.log 2>&1
cat gpurun_out/${T}_paths.log
