timeout 900 python -m pytest tests -m gpu -x -q -k "large or batched or cluster_matches" 2>&1 | tail -2
python tools/profile_case.py --config 4 --n-rods 127 --method rk4 | cut -c1-130
python tools/profile_case.py --config 4 --n-rods 127 --method sp6 | cut -c1-130
python tools/profile_case.py --config 4 --n-rods 255 --method rk4 | cut -c1-130
