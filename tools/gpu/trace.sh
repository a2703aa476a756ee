# CTA-0 event timelines of chosen ResNet-50 layers (libdg_trace.so, -DDG_TRACE)
mkdir -p gpurun_out/r2
for l in ${LAYERS:-2 1 28 15 10}; do
  echo "=== conv$l"; timeout 120 python tools/trace_ts.py conv$l --short 2>&1 | tail -80
done > gpurun_out/r2/${TAG:-trace}.log 2>&1
tail -5 gpurun_out/r2/${TAG:-trace}.log
