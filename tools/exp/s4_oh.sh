mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "onehot" > gpurun_out/s4/tests_oh.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_oh.txt
timeout -s KILL 200 python tools/time_gemm.py --shapes 4096x4096x4096,8192x8192x8192 --variants cc,prepared,onehot,f4 --iters 5 > gpurun_out/s4/time_oh.txt 2>&1
