mkdir -p gpurun_out/s4
L=24,28,31,42,43,44,45,46,47,48,49
DG_EXP_U12=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv or prepared" > gpurun_out/s4/tests_u12b.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_u12b.txt
DG_EXP_U12=1 timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_u12b.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_u8b.txt 2>&1
DG_EXP_U12=1 timeout -s KILL 200 python tools/time_gemm.py --shapes 8192x8192x8192,16384x16384x16384 --variants prepared --iters 5 > gpurun_out/s4/time_u12.txt 2>&1
