mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01u_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r01u_gpu_tests.log
tail -3 gpurun_out/r01u_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01u_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r01u_smoke.log; tail -3 gpurun_out/r01u_smoke.log
timeout 600 python bench.py > gpurun_out/r01u_bench.json 2> gpurun_out/r01u_bench.err
cut -c1-200 gpurun_out/r01u_bench.json
