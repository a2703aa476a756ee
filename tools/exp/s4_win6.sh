mkdir -p gpurun_out/s4
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/s4/tests_win6.txt 2>&1; echo "exit $?" >> gpurun_out/s4/tests_win6.txt
timeout -s KILL 300 python bench.py > gpurun_out/s4/bench_win6.json 2> gpurun_out/s4/bench_win6.err
timeout -s KILL 200 python bench.py --workload vgg16 --steps 10 > gpurun_out/s4/bench_vgg_win6.json 2> gpurun_out/s4/bench_vgg_win6.err
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/s4/bench_r18_win6.json 2> gpurun_out/s4/bench_r18_win6.err
