# ncu --set full of the fused prolongation + coloured sweep at config 3 level 9
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:'k_cgs_cols.*Lb1E' -c 1 -f \
    -o gpurun_out/cgs_prolong_L9 python tools/cgs_prolong_time.py 9 > gpurun_out/ncu_cgs_prolong.log 2>&1
