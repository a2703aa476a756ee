# round-1 (session 4) profile refresh after the whole-warp MMA issue fix
mkdir -p gpurun_out/prof4
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/prof4/tests.txt 2>&1; echo "exit $?" >> gpurun_out/prof4/tests.txt
timeout -s KILL 300 python bench.py > gpurun_out/prof4/bench_r50.json 2> gpurun_out/prof4/bench_r50.err
timeout -s KILL 200 python bench.py --workload gemm --steps 10 > gpurun_out/prof4/bench_gemm.json 2> gpurun_out/prof4/bench_gemm.err
timeout -s KILL 200 python bench.py --workload gemm --n 8192 --steps 20 > gpurun_out/prof4/bench_gemm8192.json 2> gpurun_out/prof4/bench_gemm8192.err
timeout -s KILL 200 python bench.py --workload vgg16 --steps 10 > gpurun_out/prof4/bench_vgg.json 2> gpurun_out/prof4/bench_vgg.err
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/prof4/bench_r18.json 2> gpurun_out/prof4/bench_r18.err
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/prof4/bench_ref.json 2> gpurun_out/prof4/bench_ref.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lut_gemm_ts -c 52 --csv --log-file gpurun_out/prof4/launches_r50.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-oracle > gpurun_out/prof4/ncu_launch.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/prof4/full_l1 python tools/prof_layer.py --layers 1 --iters 1 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/prof4/full_gemm python tools/time_gemm.py --shapes 8192x8192x8192 --variants prepared --iters 1 > gpurun_out/prof4/ncu_gemm.log 2>&1
