mkdir -p gpurun_out
T=${T:-r02q}
L=$PWD/paper_2306_00271_b200
timeout 900 python -m pytest tests/test_gpu_rinit.py tests/test_cpp_api.py tests/test_gpu_parity.py -m gpu -q -x -k "rinit or r_init or cpp or bulk or solve_proposed or zero" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -15 gpurun_out/${T}_tests.log
timeout 300 oracle/_ref/tests/adapter_b200 > gpurun_out/${T}_adapter.log 2>&1; echo rc=$? >> gpurun_out/${T}_adapter.log; tail -5 gpurun_out/${T}_adapter.log
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -3 gpurun_out/${T}_prof_cfg3.log
