timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ab.sh libmanybeam_b200_base.so libmanybeam_b200_opt.so 3 | head -4
bash tools/gpu/ab.sh libmanybeam_b200_base.so libmanybeam_b200_opt.so 1 | head -2
