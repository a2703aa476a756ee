mkdir -p gpurun_out/s4
L=24,28,31,42,43,45,46,48,49,51
DG_EXP_CS2=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv or prepared or gemm_random" > gpurun_out/s4/tests_cs256.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_cs256.txt
DG_EXP_CS2=1 timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_cs256.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_cs1_256.txt 2>&1
DG_EXP_CS2=1 timeout -s KILL 200 python tools/time_gemm.py --shapes 8192x8192x8192,16384x16384x16384 --variants prepared --iters 5 > gpurun_out/s4/time_cs256.txt 2>&1
