out=gpurun_out/r02_v3
mkdir -p $out
timeout 600 python -m pytest tests/test_packinfo_gpu.py tests/test_cpp_api.py tests/test_overlap_gpu.py tests/test_fused_gpu.py -x -q > $out/pytest.log 2>&1
timeout 600 python bench.py --no-configs --no-cpu > $out/bench.json 2> $out/bench.err
timeout 300 python tools/vcycle_once.py --level 10 --cycles 3 > $out/vcycle_once.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/vcycle_launches.csv \
   python tools/vcycle_once.py --level 10 --cycles 1 > $out/ncu_vc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $out/kernels_L10_times.csv python tools/kernels_once.py 10 > $out/ncu_k.log 2>&1
