mkdir -p gpurun_out/s4
DG_WIN=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,11,24,27 --iters 5 > gpurun_out/s4/prof_win.txt 2>&1
timeout -s KILL 120 python tools/prof_layer.py --layers 1,4,11,24,27 --iters 5 > gpurun_out/s4/prof_nowin.txt 2>&1
DG_WIN=1 timeout -s KILL 120 python tools/trace_ts.py conv1 --win > gpurun_out/s4/trace_win1.txt 2>&1
