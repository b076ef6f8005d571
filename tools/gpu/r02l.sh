mkdir -p gpurun_out
T=${T:-r02l}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 900 python tools/cmp_paths.py 127,255 rk4 2 > gpurun_out/${T}_paths.log 2>&1; cat gpurun_out/${T}_paths.log
timeout 900 python tools/sweep.py --cases 4 --n4 15,31,63,127,255 --reps 1 > gpurun_out/${T}_sweep4.jsonl 2> gpurun_out/${T}_sweep4.err; tail -c 600 gpurun_out/${T}_sweep4.jsonl
