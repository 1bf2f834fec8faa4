#!/bin/bash
# ncu --set full of one coloured-GS face launch (config 3 mesh) at the given levels
for L in ${LEVELS:-9}; do
  ncu --set full --import-source on --clock-control none -k regex:k_cgs_duo -c 1 -f -o gpurun_out/cgs_duo_L$L \
      python tools/smoother_time.py cgs $L 1 > gpurun_out/ncu_cgs_L$L.log 2>&1
done
