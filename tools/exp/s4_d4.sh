mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm4 or conv4 or digits4" > gpurun_out/s4/tests_d4.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_d4.txt
