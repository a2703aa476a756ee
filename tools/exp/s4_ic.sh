mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv" > gpurun_out/s4/tests_ic.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_ic.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 1,3,4,11,13,23,24,45,46 --iters 5 > gpurun_out/s4/prof_ic.txt 2>&1
DG_NO_TMAIC=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,3,4,11,13,23,24,45,46 --iters 5 > gpurun_out/s4/prof_noic.txt 2>&1
