mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/final/tests.txt 2>&1; echo "exit $?" >> gpurun_out/final/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "exit $?" >> gpurun_out/final/smoke.txt
timeout -s KILL 300 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
