# Round-2 final validation of HEAD on one B200: full GPU test suite, smoke,
# bench line + reference arm, launch list, ncu --set full of the cfg3 kernel,
# cfg4 sweep with clocks, full-size parity against the reference build.
mkdir -p gpurun_out
T=${T:-r02x}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/${T}_smoke.log; tail -3 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cut -c1-300 gpurun_out/${T}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
cut -c1-300 gpurun_out/${T}_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --legs '' > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:cluster_kernel -c 1 -f -o gpurun_out/${T}_cfg3 python tools/profile_case.py --config 3 > gpurun_out/${T}_ncu_cfg3.log 2>&1
tail -2 gpurun_out/${T}_ncu_cfg3.log
timeout 1200 python tools/sweep.py --cases 4 --n4 15,31,63,127,255 --reps 1 > gpurun_out/${T}_sweep4.jsonl 2> gpurun_out/${T}_sweep4.err; tail -c 400 gpurun_out/${T}_sweep4.jsonl
timeout 1500 python tools/parity_full.py --noise --out gpurun_out/${T}_parity.json > gpurun_out/${T}_parity.log 2>&1; tail -5 gpurun_out/${T}_parity.log
ls gpurun_out | grep ${T}
