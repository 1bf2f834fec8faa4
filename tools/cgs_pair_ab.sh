# coloured-GS sweep pairs: per-level sweep times for the pair variants (HYB_CGS_CFG)
out=gpurun_out/cgs_pair_ab.txt
: > $out
for v in 0 21 22; do
  echo "== HYB_CGS_CFG $v" >> $out
  for L in 8 9; do HYB_CGS_CFG=$v timeout 300 python tools/cgs_pair_time.py $L >> $out 2>&1; done
done
HYB_CGS_CFG=21 timeout 900 python -m pytest tests/test_cgs_pair_gpu.py -x -q 2>&1 | tail -3 >> $out
