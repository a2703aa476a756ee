timeout -s KILL 120 python tools/prof_layer.py --layers 1,15,28,47 --iters 3 > gpurun_out/exp16.txt 2>&1
echo == NO_WIN >> gpurun_out/exp16.txt
DG_NO_WIN=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,15,28,47 --iters 3 >> gpurun_out/exp16.txt 2>&1
