MB_LIB=$PWD/paper_2306_00271_b200/libmanybeam_b200_prof.so python tools/profile_case.py --config 1 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "not cluster and not cooperative and not large and not batched" 2>&1 | tail -2
for c in 1 2; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-120; done
