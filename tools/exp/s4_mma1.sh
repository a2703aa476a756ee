mkdir -p gpurun_out/s4
timeout -s KILL 120 python tools/prof_layer.py --layers 0,1,2,3,11,23,27,45 --iters 5 > gpurun_out/s4/prof_mma1.txt 2>&1
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/s4/tests_mma1.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_mma1.txt
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_r50_mma1.json 2> gpurun_out/s4/bench_r50_mma1.err
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/s4/bench_gemm_mma1.json 2>&1
