out=gpurun_out/mega_ab.txt
: > $out
for n in 4 8 16 32 64; do
  for d in 16384 4096; do
    echo "max_n $n dofs/cta $d: $(HYB_MEGA_MAXN=$n HYB_MEGA_DPC=$d python tools/mega_time.py 2>&1 | tail -1)" >> $out
  done
done
