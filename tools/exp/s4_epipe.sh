mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s4/tests_epipe.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_epipe.txt
L=2,3,4,6,12,13,16,25,29,44,45
timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_epipe.txt 2>&1
DG_NO_EPIPIPE=1 timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_noepipe.txt 2>&1
