mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01ab_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r01ab_gpu_tests.log
tail -3 gpurun_out/r01ab_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01ab_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r01ab_smoke.log; tail -2 gpurun_out/r01ab_smoke.log
timeout 600 python bench.py > gpurun_out/r01ab_bench.json 2> gpurun_out/r01ab_bench.err
cut -c1-200 gpurun_out/r01ab_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01ab_reference.json 2> gpurun_out/r01ab_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01ab_launches_bench_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01ab_ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:propagate_kernel -c 1 -f -o gpurun_out/r01ab_cfg1 python tools/profile_case.py --config 1 > gpurun_out/r01ab_ncu_cfg1.log 2>&1
python tools/sweep.py --cases 0,1,2,4 --n4 15,31,63 --reps 2 > gpurun_out/sweep_r01ab_small.jsonl 2> gpurun_out/sweep_r01ab_small.err
ls gpurun_out | grep r01ab
