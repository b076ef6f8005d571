mkdir -p gpurun_out
T=r02f
L=$PWD/paper_2306_00271_b200
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -5 gpurun_out/${T}_gpu_tests.log
timeout 300 python tools/cfg3_accuracy.py run --role dev3m --out gpurun_out/${T}_acc_dev3m.npz > /dev/null 2>&1
timeout 300 python tools/cfg3_accuracy.py run --role dev3m_nofsal --out gpurun_out/${T}_acc_nofsal.npz > /dev/null 2>&1
timeout 300 python tools/cfg3_accuracy.py run --role devpath2 --out gpurun_out/${T}_acc_p2.npz > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cut -c1-300 gpurun_out/${T}_bench.json
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -1 gpurun_out/${T}_prof_cfg3.log
ls gpurun_out | grep ${T}
