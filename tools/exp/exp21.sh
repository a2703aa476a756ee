timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp21_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp21_tests.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 1,11,13,15,24,28,43,47 --iters 3 > gpurun_out/exp21.txt 2>&1
