mkdir -p gpurun_out/s4
DG_EXP_CS2=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s4/tests_cs2.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_cs2.txt
DG_EXP_CS2=1 timeout -s KILL 120 python tools/prof_layer.py --layers 0,2,3,5,10,11,12,14 --iters 5 > gpurun_out/s4/prof_cs2.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 0,2,3,5,10,11,12,14 --iters 5 > gpurun_out/s4/prof_cs1.txt 2>&1
