# Round profiling: bench lines (N=1), ncu launch list of one ResNet-50 step, full ncu of two layers.
mkdir -p gpurun_out/prof
timeout -s KILL 300 python bench.py > gpurun_out/prof/bench_r50.json 2> gpurun_out/prof/bench_r50.err
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/prof/bench_gemm.json 2> gpurun_out/prof/bench_gemm.err
timeout -s KILL 200 python bench.py --workload vgg16 --steps 10 > gpurun_out/prof/bench_vgg.json 2> gpurun_out/prof/bench_vgg.err
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/prof/bench_r18.json 2> gpurun_out/prof/bench_r18.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lut_gemm_ts -c 52 --csv --log-file gpurun_out/prof/launches_r50.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-oracle > gpurun_out/prof/ncu_launch.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/prof/full_l28 python tools/prof_layer.py --layers 28 --iters 1 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/prof/full_l2 python tools/prof_layer.py --layers 2 --iters 1 > /dev/null 2>&1
