mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "f4" > gpurun_out/s4/tests_f4.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_f4.txt
timeout -s KILL 200 python tools/time_gemm.py --shapes 4096x4096x4096,8192x8192x8192,16384x16384x16384 --variants prepared,f4 --iters 5 > gpurun_out/s4/time_f4.txt 2>&1
