# session-4 re-entry check: GPU tests + bench lines on the restored tree
mkdir -p gpurun_out/s4
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/s4/tests.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests.txt
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_r50.json 2> gpurun_out/s4/bench_r50.err
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/s4/bench_gemm.json 2> gpurun_out/s4/bench_gemm.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4/smoke.txt 2>&1; echo "exit $?" >> gpurun_out/s4/smoke.txt
