out=gpurun_out/jacobi2_ab.txt
: > $out
python -m pytest tests/test_jacobi2_gpu.py tests/test_parity_gpu.py tests/test_configs_gpu.py -x -q 2>&1 | tail -3 >> $out
echo "vcycle default: $(python tools/vcycle_once.py --level 10 --cycles 10 2>&1 | tail -1)" >> $out
