mkdir -p gpurun_out/s4
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/s4/tests_gf.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_gf.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 1,3,4,11,23,27,45 --iters 5 > gpurun_out/s4/prof_gf.txt 2>&1
DG_NO_GFAST=1 timeout -s KILL 120 python tools/prof_layer.py --layers 1,3,4,11,23,27,45 --iters 5 > gpurun_out/s4/prof_nogf.txt 2>&1
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_r50_gf.json 2> gpurun_out/s4/bench_r50_gf.err
