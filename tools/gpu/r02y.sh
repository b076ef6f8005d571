mkdir -p gpurun_out
T=${T:-r02y}
timeout 1500 python -m pytest tests -m gpu -q -k "bulk or r_init or rinit or cpp or large_path or n255 or golden" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -5 gpurun_out/${T}_tests.log
grep -E "^E  |FAILED|solve_proposed:" gpurun_out/${T}_tests.log | head -30
timeout 300 python tools/cmp_paths.py 127 rk4 2
