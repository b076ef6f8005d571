mkdir -p gpurun_out
for P in 2 3 4; do echo parts=$P; MB_BIG_PARTS=$P timeout 600 python tools/cmp_paths.py 127,255 rk4 2; done
MB_BIG_PARTS=4 timeout 900 python -m pytest tests -m gpu -q -x -k "large_path or n255 or batched or two_streams" 2>&1 | tail -3
