timeout 600 ncu --set full --import-source on --clock-control none -k regex:big_gj --launch-skip 20 -c 3 -f -o gpurun_out/r01m_gj python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 50 --z-bottom -0.8 > gpurun_out/ncu_gj.log 2>&1
tail -2 gpurun_out/ncu_gj.log
