mkdir -p gpurun_out
T=${T:-r02g}
L=$PWD/paper_2306_00271_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 600 python bench.py --legs '1' --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cut -c1-300 gpurun_out/${T}_bench.json
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -1 gpurun_out/${T}_prof_cfg3.log
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 1 > gpurun_out/${T}_prof_cfg1.log 2>&1
tail -1 gpurun_out/${T}_prof_cfg1.log
timeout 300 python tools/cfg3_accuracy.py run --role dev3m --out gpurun_out/${T}_acc_dev3m.npz > /dev/null 2>&1
