mkdir -p gpurun_out/r2
TRACE_STAGES=${TRACE_STAGES:-96} timeout 300 python tools/trace_ts.py ${SHAPE:-16384x16384x16384} --short > gpurun_out/r2/${TAG}_trace.log 2>&1
tail -60 gpurun_out/r2/${TAG}_trace.log
