timeout 900 python -m pytest tests -m gpu -x -q -k "not cluster and not cooperative and not large and not batched" 2>&1 | tail -2
bash tools/gpu/ab.sh libmanybeam_b200_base.so libmanybeam_b200_opt.so 1 | head -4
bash tools/gpu/ab.sh libmanybeam_b200_base.so libmanybeam_b200_opt.so 2 | head -4
