mkdir -p gpurun_out/s4
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/s4/tests_walk.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_walk.txt
timeout -s KILL 120 python tools/prof_layer.py --layers 0,2,4,11,24,28,42,43,45 --iters 5 > gpurun_out/s4/prof_walk.txt 2>&1
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_walk.json 2> gpurun_out/s4/bench_walk.err
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/s4/bench_gemm_walk.json 2> gpurun_out/s4/bench_gemm_walk.err
timeout -s KILL 200 python bench.py --workload vgg16 --steps 10 > gpurun_out/s4/bench_vgg_walk.json 2> gpurun_out/s4/bench_vgg_walk.err
