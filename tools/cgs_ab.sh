# A/B of the small-face coloured-GS kernels (HYB_CGS_CFG=12: the row-block kernel) on config 3's mesh
out=gpurun_out/cgs_ab.txt
: > $out
for L in 4 5 6 7; do
  echo "L$L old: $(HYB_CGS_CFG=12 python tools/smoother_time.py cgs $L 20 2>&1 | tail -3 | tr '\n' ' ')" >> $out
  echo "L$L new: $(python tools/smoother_time.py cgs $L 20 2>&1 | tail -3 | tr '\n' ' ')" >> $out
done
python -m pytest tests/test_configs_gpu.py -x -q -k "colored" 2>&1 | tail -3 >> $out
echo "cycle new: $(python tools/vcycle_once.py --mesh cfg3 --level 9 --smoother colored_gs --nu 3 3 --cycles 3 2>&1 | tail -1)" >> $out
echo "cycle old: $(HYB_CGS_CFG=12 python tools/vcycle_once.py --mesh cfg3 --level 9 --smoother colored_gs --nu 3 3 --cycles 3 2>&1 | tail -1)" >> $out
