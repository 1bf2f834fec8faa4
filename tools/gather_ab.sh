# sorted ghost refresh: parity tests that exercise it, the level-9 gather under ncu, config-3 cycle, bench
out=gpurun_out/gather_ab.txt
: > $out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_overlap_gpu.py tests/test_sync_directions_gpu.py tests/test_mega_gpu.py tests/test_cgs_pair_gpu.py -x -q 2>&1 | tail -3 >> $out
timeout 300 python tools/cfg3_profile.py 9 >> $out 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-configs >> $out 2>&1
bash tools/ncu_gather.sh
