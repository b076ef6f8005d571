mkdir -p gpurun_out
T=${T:-r02z}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_gpu_tests.log
tail -4 gpurun_out/${T}_gpu_tests.log
grep -E "^E  |FAILED|solve_proposed:" gpurun_out/${T}_gpu_tests.log | head -30
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/${T}_smoke.log; tail -2 gpurun_out/${T}_smoke.log
timeout 300 oracle/_ref/tests/adapter_b200 > gpurun_out/${T}_adapter.log 2>&1; echo rc=$? >> gpurun_out/${T}_adapter.log; tail -3 gpurun_out/${T}_adapter.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; cut -c1-200 gpurun_out/${T}_bench.json
