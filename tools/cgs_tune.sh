#!/bin/bash
# coloured-GS face kernel variants (HYB_CGS_CFG, see launch_cgs_faces_cols) on config 3's mesh
for cfg in ${CFGS:-0 1 2 3}; do
  for L in ${LEVELS:-9 8 7}; do
    HYB_CGS_CFG=$cfg python tools/smoother_time.py cgs $L 10 > /tmp/st.txt 2>&1
    echo "cfg $cfg: $(head -1 /tmp/st.txt)"
  done
done
