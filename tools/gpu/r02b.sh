mkdir -p gpurun_out
T=r02b
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/${T}_smoke.log; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cut -c1-400 gpurun_out/${T}_bench.json
# phase profile of cfg3 (instrumented build)
MB_LIB=$PWD/paper_2306_00271_b200/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 > gpurun_out/${T}_prof_cfg3.log 2>&1
tail -2 gpurun_out/${T}_prof_cfg3.log
MB_LIB=$PWD/paper_2306_00271_b200/libmanybeam_b200_prof.so timeout 300 python tools/profile_case.py --config 3 --path 3 > gpurun_out/${T}_prof_cfg3_p3.log 2>&1
tail -2 gpurun_out/${T}_prof_cfg3_p3.log
# cfg3 accuracy: the three device designs on the full workload
for r in dev3m devpath2 devpath3; do
  timeout 600 python tools/cfg3_accuracy.py run --role $r --out gpurun_out/${T}_acc_$r.npz > gpurun_out/${T}_acc_$r.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --legs '' > gpurun_out/${T}_ncu_launch.log 2>&1
ls gpurun_out | grep ${T}
