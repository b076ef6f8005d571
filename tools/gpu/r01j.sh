mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01j_tests.log 2>&1; echo rc=$? >> gpurun_out/r01j_tests.log
tail -3 gpurun_out/r01j_tests.log
for c in 1 2; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-140; done
python tools/profile_case.py --config 4 --n-rods 63 --method rk4 | cut -c1-140
python tools/profile_case.py --config 4 --n-rods 63 --method sp6 | cut -c1-140
