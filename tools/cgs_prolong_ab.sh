out=gpurun_out/cgs_prolong_ab.txt
: > $out
for L in 8 9; do timeout 300 python tools/cgs_prolong_time.py $L >> $out 2>&1; done
