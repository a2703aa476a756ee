mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv" > gpurun_out/s4/tests_ic2.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_ic2.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,11,13,23,24,45,46 --iters 5 > gpurun_out/s4/prof_ic2.txt 2>&1
timeout -s KILL 120 python tools/trace_ts.py conv1 --win > gpurun_out/s4/trace6_conv1.txt 2>&1
