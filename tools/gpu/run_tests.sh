# GPU test + bench driver for gpurun (args: pytest selection, bench args)
set -x
mkdir -p gpurun_out/r2
nproc
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q --durations=10 ${PYTEST_SEL:-} > gpurun_out/r2/${TAG:-t}_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/r2/${TAG:-t}_pytest.log
if [ -n "${BENCH:-1}" ]; then
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/r2/${TAG:-t}_bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/r2/${TAG:-t}_bench.log | cut -c1-6000
fi
