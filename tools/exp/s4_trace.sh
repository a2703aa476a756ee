mkdir -p gpurun_out/s4
for L in 1 2 0 23; do timeout -s KILL 120 python tools/trace_ts.py conv$L --short > gpurun_out/s4/trace_conv$L.txt 2>&1; done
timeout -s KILL 120 python tools/prof_layer.py --layers 0,1,2,3,23 --iters 5 > gpurun_out/s4/prof_layers.txt 2>&1
