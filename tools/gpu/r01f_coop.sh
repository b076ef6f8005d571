mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "bulk or cluster or cooperative or golden or large" > gpurun_out/r01f_tests.log 2>&1; echo rc=$? >> gpurun_out/r01f_tests.log
tail -5 gpurun_out/r01f_tests.log
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/r01f_cfg3.json 2> gpurun_out/r01f_cfg3.err
cut -c1-400 gpurun_out/r01f_cfg3.json; tail -3 gpurun_out/r01f_cfg3.err
