timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp24_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp24_tests.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 0,2,3,12,16 --iters 3 > gpurun_out/exp24.txt 2>&1
