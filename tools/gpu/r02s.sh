mkdir -p gpurun_out
T=${T:-r02s}
for i in 1 2; do timeout 300 python bench.py --config 3 --legs '' --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3', round(d['value'],2), round(d['roofline']['frac'],4), d['clocks'])"; done
timeout 1500 python -m pytest tests -m gpu -q -x -k "config3 or cfg3 or cluster or cooperative or bulk or n255 or large_path or golden or fsal or r_init or rinit" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
grep -E "FAIL|Error|assert" gpurun_out/${T}_tests.log | head -20
