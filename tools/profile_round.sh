#!/bin/bash
# One GPU-box pass that produces a round's profile set under gpurun_out/$1:
# the bench line (and the reference arm), the bench's ncu launch list, one
# `ncu --set full` capture of the config-2 hot kernels and of the config-3
# coloured sweep, the other configurations' timings and the GPU test log.
# Each ncu command runs after the same program has exited 0 without ncu.
set -u
out=gpurun_out/${1:-prof}
mkdir -p "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$out/smi.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -q > "$out/pytest_gpu.log" 2>&1; echo "pytest_exit=$?" >> "$out/pytest_gpu.log"
timeout 900 python bench.py > "$out/bench.json" 2> "$out/bench.err"; echo "bench_exit=$?" >> "$out/bench.err"
timeout 900 python bench.py --impl reference > "$out/bench_ref.json" 2> "$out/bench_ref.err"
timeout 900 python tools/configs_time.py > "$out/configs_time.jsonl" 2> "$out/configs_time.err"
# graph-replayed cycles (five after three warm-ups) and config 3's cycle by operation
{ timeout 300 python tools/cfg3_cycles.py 9; timeout 300 python tools/jac_cycles.py cfg2; timeout 300 python tools/jac_cycles.py faces8192; } > "$out/cycles.txt" 2>&1
timeout 300 python tools/cfg3_profile.py > "$out/cfg3_profile.txt" 2>&1
if timeout 600 python bench.py --steps 2 --warmup 1 > "$out/bench_short.json" 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file "$out/bench_launches.csv" python bench.py --steps 2 --warmup 1 > "$out/ncu_launches.log" 2>&1
fi
if timeout 300 python tools/kernels_once.py 10 > "$out/kernels_once.log" 2>&1; then
  timeout 1200 ncu --set full --import-source on --clock-control none -o "$out/kernels_L10" \
    python tools/kernels_once.py 10 > "$out/ncu_kernels.log" 2>&1
fi
if timeout 300 python tools/smoother_time.py cgs 9 1 > "$out/cgs_once.log" 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cgs_duo -s 1 -c 1 -o "$out/cgs_L9" \
    python tools/smoother_time.py cgs 9 1 > "$out/ncu_cgs.log" 2>&1
fi
# the reports stay on the box; their tables come back (gpurun copies <= 64 MiB)
for rep in "$out"/*.ncu-rep; do
  [ -f "$rep" ] || continue
  base="${rep%.ncu-rep}"
  python tools/ncu_table.py "$rep" "$base.csv" --note "$(basename "$rep")" > /dev/null 2>&1
  ncu -i "$rep" --page raw --csv > "$base.raw.csv" 2> /dev/null
  ncu -i "$rep" --page source --csv --print-source sass > "$base.sass.csv" 2> /dev/null
  python tools/sass_hot.py "$base.sass.csv" 40 > "$base.sass_hot.txt" 2> /dev/null
  rm -f "$base.sass.csv"
  [ "$(stat -c %s "$rep")" -lt 20000000 ] || rm -f "$rep"
done
du -sh "$out" > "$out/du.txt"
echo done > "$out/DONE"
