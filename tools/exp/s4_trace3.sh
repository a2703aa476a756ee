mkdir -p gpurun_out/s4
for L in 1 2 0; do timeout -s KILL 120 python tools/trace_ts.py conv$L --win > gpurun_out/s4/trace3_conv$L.txt 2>&1; done
