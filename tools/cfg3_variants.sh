for v in "" "HYB_COARSE_GRID_MIN=5121"; do
  echo "== $v"; env $v python tools/vcycle_once.py --mesh cfg3 --level 9 --smoother colored_gs --nu 3 3 --cycles 5
done
python tools/smoother_time.py cgs 7 10
python tools/smoother_time.py cgs 6 10
