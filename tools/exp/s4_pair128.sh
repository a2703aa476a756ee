mkdir -p gpurun_out/s4
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window or conv" > gpurun_out/s4/tests_p128.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_p128.txt
timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 1,2 --iters 5 > gpurun_out/s4/prof_p128.txt 2>&1
DG_NO_WPAIR=1 timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 1,2 --iters 5 > gpurun_out/s4/prof_nop128.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,15 --iters 5 >> gpurun_out/s4/prof_p128.txt 2>&1
DG_NO_WPAIR=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,15 --iters 5 >> gpurun_out/s4/prof_nop128.txt 2>&1
