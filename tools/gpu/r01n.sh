mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r01n_bench.json 2> gpurun_out/r01n_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01n_reference.json 2> gpurun_out/r01n_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01n_launches_bench_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01n_ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:propagate_kernel -c 1 -f -o gpurun_out/r01n_cfg1 python tools/profile_case.py --config 1 > gpurun_out/r01n_ncu_cfg1.log 2>&1
cut -c1-300 gpurun_out/r01n_bench.json; cut -c1-200 gpurun_out/r01n_reference.json
