mkdir -p gpurun_out/s4
DG_EXP_U12=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv" > gpurun_out/s4/tests_u12.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_u12.txt
DG_EXP_U12=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,7 --iters 5 > gpurun_out/s4/prof_u12.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,7 --iters 5 > gpurun_out/s4/prof_u8.txt 2>&1
