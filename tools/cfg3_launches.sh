# launch list of config 3's V(3,3) cycle (one warm-up + one profiled cycle; graphs replay kernels the same)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg3_launches.csv \
    python tools/vcycle_once.py --mesh cfg3 --level 9 --smoother colored_gs --nu 3 3 --cycles 1 > gpurun_out/cfg3_launches.log 2>&1
