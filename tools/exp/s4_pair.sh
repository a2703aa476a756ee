mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window or conv" > gpurun_out/s4/tests_pair.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_pair.txt
timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 1 --iters 5 > gpurun_out/s4/prof_pair.txt 2>&1
DG_NO_WPAIR=1 timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 1 --iters 5 > gpurun_out/s4/prof_nopair.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,5 --iters 5 >> gpurun_out/s4/prof_pair.txt 2>&1
DG_NO_WPAIR=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,5 --iters 5 >> gpurun_out/s4/prof_nopair.txt 2>&1
