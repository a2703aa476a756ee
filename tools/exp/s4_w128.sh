mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window or conv" > gpurun_out/s4/tests_w128.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_w128.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 15,18,21 --iters 5 > gpurun_out/s4/prof_w128.txt 2>&1
DG_NO_WIN128=1 timeout -s KILL 120 python tools/prof_layer.py --layers 15,18,21 --iters 5 > gpurun_out/s4/prof_now128.txt 2>&1
