mkdir -p gpurun_out/s4
timeout -s KILL 120 python tools/prof_layer.py --layers 0,1,2,3,11,23,27,45 --iters 5 > gpurun_out/s4/prof_stage.txt 2>&1
timeout -s KILL 120 python tools/trace_ts.py conv1 --win > gpurun_out/s4/trace4_conv1.txt 2>&1
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/s4/bench_gemm_stage.json 2>&1
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_r50_stage.json 2> gpurun_out/s4/bench_r50_stage.err
