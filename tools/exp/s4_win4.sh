mkdir -p gpurun_out/s4
DG_WIN=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window" > gpurun_out/s4/tests_win4.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_win4.txt
DG_WIN=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,5,8 --iters 5 > gpurun_out/s4/prof_win4.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,5,8 --iters 5 > gpurun_out/s4/prof_nowin4.txt 2>&1
DG_WIN=1 timeout -s KILL 120 python tools/trace_ts.py conv1 --win > gpurun_out/s4/trace_win4.txt 2>&1
