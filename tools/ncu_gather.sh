# ncu --set full of the largest ghost gather launch of a config-3 level-9 sweep
ncu --set full --clock-control none -k regex:k_ghost_gather4 --launch-skip 2 -c 1 -f -o gpurun_out/gather_L9 \
    python tools/smoother_time.py cgs 9 2 > gpurun_out/ncu_gather.log 2>&1
