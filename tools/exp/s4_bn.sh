mkdir -p gpurun_out/s4
L=24,28,31,42,43,44,45,46,47,48,49,50,51
DG_TS_NO_BN256=1 timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_nobn256.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_bn256.txt 2>&1
