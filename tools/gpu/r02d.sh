mkdir -p gpurun_out
T=r02d
L=$PWD/paper_2306_00271_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 600 python bench.py --legs '1' --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cut -c1-300 gpurun_out/${T}_bench.json
MB_LIB=$L/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -1 gpurun_out/${T}_prof_cfg3.log
timeout 300 python tools/cfg3_accuracy.py run --role dev3m --out gpurun_out/${T}_acc_dev3m.npz > /dev/null 2>&1
MB_LIB=$L/libmanybeam_b200_exact.so timeout 300 python tools/cfg3_accuracy.py run --role dev3m --out gpurun_out/${T}_acc_exact.npz > /dev/null 2>&1
MB_LIB=$L/libmanybeam_b200_nofma.so timeout 300 python tools/cfg3_accuracy.py run --role dev3m --out gpurun_out/${T}_acc_nofma.npz > /dev/null 2>&1
MB_LIB=$L/libmanybeam_b200_nofma.so timeout 300 python tools/cfg3_accuracy.py run --role dev3m_nofsal --out gpurun_out/${T}_acc_nofma_nofsal.npz > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cluster_kernel -c 1 -f -o gpurun_out/${T}_cfg3 python tools/profile_case.py --config 3 > gpurun_out/${T}_ncu_cfg3.log 2>&1
tail -2 gpurun_out/${T}_ncu_cfg3.log
ls gpurun_out | grep ${T}
