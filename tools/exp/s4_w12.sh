mkdir -p gpurun_out/s4
DG_EXP_WIN12=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window" > gpurun_out/s4/tests_w12.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_w12.txt
DG_EXP_WIN12=1 timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 1,2 --iters 5 > gpurun_out/s4/prof_w12.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 1,2 --iters 5 > gpurun_out/s4/prof_w8.txt 2>&1
DG_EXP_WIN12=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,5,8 --iters 5 >> gpurun_out/s4/prof_w12.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,5,8 --iters 5 >> gpurun_out/s4/prof_w8.txt 2>&1
