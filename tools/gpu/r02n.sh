mkdir -p gpurun_out
T=${T:-r02n}
L=$PWD/paper_2306_00271_b200
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -2 gpurun_out/${T}_prof_cfg3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c4n127rk4.csv python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 40 > /dev/null 2>&1
python tools/ncu_summary.py ${T}_c4n127 /dev/null gpurun_out/${T}_launches_c4n127rk4.csv 2>&1 | tail -30
