timeout 900 python -m pytest tests -m gpu -x -q -k "large or batched or golden or cluster_matches or fullsize" 2>&1 | tail -2
for L in libmanybeam_b200_base.so libmanybeam_b200_opt.so; do for n in "127 rk4" "127 sp6"; do set -- $n; echo -n "$L $1 $2 "; MB_LIB=$PWD/paper_2306_00271_b200/$L python tools/profile_case.py --config 4 --n-rods $1 --method $2 | cut -c1-90; done; done
