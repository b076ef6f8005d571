mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01h_tests.log 2>&1; echo rc=$? >> gpurun_out/r01h_tests.log
tail -3 gpurun_out/r01h_tests.log
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/r01h_cfg3.json 2> gpurun_out/r01h_cfg3.err
cut -c1-300 gpurun_out/r01h_cfg3.json
timeout 600 python tools/cmp_paths.py 127,255 sp6 0,3,4 2>&1 | tail -8
