timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp29_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp29_tests.txt
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/exp29_r18.json 2>&1
timeout -s KILL 120 python tools/prof_r18.py > gpurun_out/exp29_r18layers.txt 2>&1
timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp29_r50.json 2>&1
