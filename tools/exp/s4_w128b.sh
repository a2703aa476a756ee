mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window or conv" > gpurun_out/s4/tests_w128b.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_w128b.txt
timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 3 --iters 5 > gpurun_out/s4/prof_w128b.txt 2>&1
DG_NO_WIN128=1 timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 3 --iters 5 > gpurun_out/s4/prof_now128b.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 15 --iters 5 >> gpurun_out/s4/prof_w128b.txt 2>&1
