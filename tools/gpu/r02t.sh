mkdir -p gpurun_out
T=${T:-r02t}
L=$PWD/paper_2306_00271_b200
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -2 gpurun_out/${T}_prof_cfg3.log
