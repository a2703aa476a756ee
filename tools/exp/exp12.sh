for l in 1 12; do echo "== vgg layer $l"; timeout -s KILL 60 python tools/prof_layer.py --cfg 4 --batch 64 --layers $l --iters 2 2>&1 | tail -1; done > gpurun_out/exp12.txt 2>&1
timeout -s KILL 300 python -m pytest tests -m gpu -x -q > gpurun_out/exp12_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp12_tests.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 0,1,2,4,10,11,12,13,14,16,24,25,27,28,43,44,47 --iters 3 >> gpurun_out/exp12.txt 2>&1
