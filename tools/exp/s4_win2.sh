mkdir -p gpurun_out/s4
DG_WIN=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,7,11,14,17,20,24,27,30,33,36,39,43,46,49 --iters 5 > gpurun_out/s4/prof_win2.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,7,11,14,17,20,24,27,30,33,36,39,43,46,49 --iters 5 > gpurun_out/s4/prof_nowin2.txt 2>&1
