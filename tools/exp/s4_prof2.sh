# session-4 final profile refresh
mkdir -p gpurun_out/prof5
timeout -s KILL 600 python -m pytest tests -m gpu -q > gpurun_out/prof5/tests.txt 2>&1; echo "exit $?" >> gpurun_out/prof5/tests.txt
timeout -s KILL 300 python bench.py > gpurun_out/prof5/bench_r50.json 2> gpurun_out/prof5/bench_r50.err
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/prof5/bench_gemm.json 2> gpurun_out/prof5/bench_gemm.err
timeout -s KILL 200 python bench.py --workload gemm --variant f4 --steps 10 > gpurun_out/prof5/bench_gemm_f4.json 2> gpurun_out/prof5/bench_gemm_f4.err
timeout -s KILL 200 python bench.py --workload vgg16 --steps 10 > gpurun_out/prof5/bench_vgg.json 2> gpurun_out/prof5/bench_vgg.err
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/prof5/bench_r18.json 2> gpurun_out/prof5/bench_r18.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof5/launches_r50.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-oracle > gpurun_out/prof5/ncu_launch.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/prof5/full_onehot python tools/time_gemm.py --shapes 4096x4096x4096 --variants onehot --iters 1 > gpurun_out/prof5/ncu_onehot.log 2>&1
