# quick GPU check: a pytest selection + optional trace layers
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()"
if [ -n "$PYTEST_SEL" ]; then
  timeout 900 python -m pytest -m gpu -q -x ${PYTEST_SEL:-tests} > gpurun_out/r2/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2/${TAG}_pytest.log
fi
if [ -n "$LAYERS" ]; then
  for l in $LAYERS; do echo "=== conv$l"; timeout 120 python tools/trace_ts.py conv$l --short 2>&1 | tail -${TRACE_TAIL:-30}; done > gpurun_out/r2/${TAG}_trace.log 2>&1
fi
if [ -n "$PROF" ]; then
  timeout 300 python tools/prof_layer.py $PROF > gpurun_out/r2/${TAG}_prof.log 2>&1; echo "prof rc=$?"; cat gpurun_out/r2/${TAG}_prof.log | tail -60
fi
