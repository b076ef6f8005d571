mkdir -p gpurun_out
T=${T:-r02r}
L=$PWD/paper_2306_00271_b200
timeout 900 python -m pytest tests/test_gpu_rinit.py -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -5 gpurun_out/${T}_tests.log
MB_LIB=$L/libmanybeam_b200_proff.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -3 gpurun_out/${T}_prof_cfg3.log
