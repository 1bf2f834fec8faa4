# megakernel A/B: the mega tests, then cycle times for max_n x dofs-per-CTA settings
out=gpurun_out/mega_ab.txt
: > $out
python -m pytest tests/test_mega_gpu.py -x -q 2>&1 | tail -3 >> $out
for n in 16 32 64; do
  for d in 65536 16384 4096; do
    echo "max_n $n dofs/cta $d: $(HYB_MEGA_MAXN=$n HYB_MEGA_DPC=$d python tools/mega_time.py 2>&1 | tail -1)" >> $out
  done
done
