# ncu --set full of one coloured-GS pair launch and one single launch (config 3 mesh, level ${L:-9})
L=${L:-9}
ncu --set full --import-source on --clock-control none -k regex:k_cgs_pair -c 1 -f -o gpurun_out/cgs_pair_L$L \
    python tools/cgs_pair_time.py $L > gpurun_out/ncu_cgs_pair.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cgs_cols -c 1 -f -o gpurun_out/cgs_cols_L$L \
    python tools/cgs_pair_time.py $L > gpurun_out/ncu_cgs_cols.log 2>&1
