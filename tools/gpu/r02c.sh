mkdir -p gpurun_out
T=r02c
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 600 python bench.py --legs '' --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cut -c1-300 gpurun_out/${T}_bench.json
MB_LIB=$PWD/paper_2306_00271_b200/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -2 gpurun_out/${T}_prof_cfg3.log
timeout 300 python tools/profile_case.py --config 1 --reps 3 > gpurun_out/${T}_cfg1.log 2>&1; tail -1 gpurun_out/${T}_cfg1.log
