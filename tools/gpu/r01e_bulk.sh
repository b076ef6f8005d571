mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "bulk or cluster or golden" > gpurun_out/r01e_tests.log 2>&1; echo rc=$? >> gpurun_out/r01e_tests.log
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/r01e_cfg3.json 2> gpurun_out/r01e_cfg3.err
tail -5 gpurun_out/r01e_tests.log; cat gpurun_out/r01e_cfg3.json | cut -c1-300
