mkdir -p gpurun_out/s4
timeout -s KILL 200 python bench.py --workload gemm --variant f4 --steps 10 > gpurun_out/s4/bench_gemm_f4.json 2> gpurun_out/s4/bench_gemm_f4.err
timeout -s KILL 200 python bench.py --workload gemm --levels uniform --steps 10 > gpurun_out/s4/bench_gemm_uni.json 2> gpurun_out/s4/bench_gemm_uni.err
timeout -s KILL 200 python bench.py --workload gemm --n 8192 --variant f4 --steps 20 > gpurun_out/s4/bench_gemm8192_f4.json 2> gpurun_out/s4/bench_gemm8192_f4.err
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_f4 -c 1 -o gpurun_out/s4/full_f4 python tools/time_gemm.py --shapes 8192x8192x8192 --variants f4 --iters 1 > gpurun_out/s4/ncu_f4.log 2>&1
