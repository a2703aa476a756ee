mkdir -p gpurun_out/s4
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_r50_v2.json 2> gpurun_out/s4/bench_r50_v2.err
timeout -s KILL 200 python bench.py --workload vgg16 --steps 10 > gpurun_out/s4/bench_vgg_v2.json 2> gpurun_out/s4/bench_vgg_v2.err
