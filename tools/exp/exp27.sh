timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp27_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp27_tests.txt
timeout -s KILL 100 python tools/prof_layer.py --layers 2,3,12,13,16,25,29 --iters 3 > gpurun_out/exp27.txt 2>&1
