timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or cooperative or bulk" 2>&1 | tail -2
bash tools/gpu/ab.sh libmanybeam_b200_base.so libmanybeam_b200_w64.so 3 | head -4
for L in libmanybeam_b200_base.so libmanybeam_b200_w64.so; do MB_LIB=$PWD/paper_2306_00271_b200/$L python tools/profile_case.py --config 3 --path 3 | cut -c1-100; done
