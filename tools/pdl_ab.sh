# A/B of programmatic dependent launch (HYB_PDL=0 off; HYB_PDL_MAX: largest grid launched programmatically)
out=gpurun_out/pdl_ab.txt
: > $out
for cfg in "HYB_PDL=0" "HYB_PDL_MAX=1184" "HYB_PDL_MAX=300" "HYB_PDL_MAX=5000" "HYB_PDL=0" "HYB_PDL_MAX=1184"; do
  echo "$cfg cfg2 vcycle: $(env $cfg python tools/vcycle_once.py --level 10 --cycles 10 2>&1 | tail -1)" >> $out
  echo "$cfg cfg1: $(env $cfg python tools/configs_time.py --configs cfg1 2>&1 | tail -1 | cut -c60-130)" >> $out
  echo "$cfg cfg3: $(env $cfg python tools/vcycle_once.py --mesh cfg3 --level 9 --smoother colored_gs --nu 3 3 --cycles 3 2>&1 | tail -1)" >> $out
done
