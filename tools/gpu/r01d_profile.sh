mkdir -p gpurun_out
for s in 200000 160000 113000 100000; do ./tools/cluster_occ $s 4 6 7 8 9 10 12 13 14 16; done > gpurun_out/cluster_occ.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:propagate_kernel -c 1 -f -o gpurun_out/r01d_cfg1 python tools/profile_case.py --config 1 > gpurun_out/ncu_cfg1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cluster_kernel -c 1 -f -o gpurun_out/r01d_cfg3 python tools/profile_case.py --config 3 > gpurun_out/ncu_cfg3.log 2>&1
ls -la gpurun_out
