mkdir -p gpurun_out
for p in 3 4; do python tools/profile_case.py --config 3 --path $p 2>&1 | cut -c1-200; done
timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or cooperative or bulk" 2>&1 | tail -3
