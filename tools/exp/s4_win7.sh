mkdir -p gpurun_out/s4
L=28,31,34,46,49
DG_WIN=1 timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_win7.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 5 > gpurun_out/s4/prof_nowin7.txt 2>&1
DG_WIN=1 timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 3,5,8,10 --iters 5 >> gpurun_out/s4/prof_win7.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --cfg 4 --batch 64 --layers 3,5,8,10 --iters 5 >> gpurun_out/s4/prof_nowin7.txt 2>&1
