mkdir -p gpurun_out
T=${T:-r02w}
timeout 900 python tools/cmp_paths.py 127,255 rk4 2 > gpurun_out/${T}_paths.log 2>&1
cat gpurun_out/${T}_paths.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "large_path or n255 or batched or config3_subset or fsal or r_init_large" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
