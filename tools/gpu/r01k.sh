mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or cooperative or bulk or golden or large" 2>&1 | tail -2
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-140
python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 50 --z-bottom -0.8 | cut -c1-150
timeout 600 ncu --set full --import-source on --clock-control none -k regex:big_stage --launch-skip 40 -c 4 -f -o gpurun_out/r01k_c4n127rk4 python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 50 --z-bottom -0.8 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01k_launches_c4n127rk4.csv python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 50 --z-bottom -0.8 > /dev/null 2>&1
tail -2 gpurun_out/ncu_c4.log
