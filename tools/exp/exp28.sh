timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp28_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp28_tests.txt
timeout -s KILL 100 python tools/prof_layer.py --layers 0,4,10,2 --iters 3 > gpurun_out/exp28.txt 2>&1
echo == NO_ASM >> gpurun_out/exp28.txt
DG_NO_ASM=1 timeout -s KILL 100 python tools/prof_layer.py --layers 0,4,10,2 --iters 3 >> gpurun_out/exp28.txt 2>&1
timeout -s KILL 200 python bench.py --e2e-steps 0 --no-oracle > gpurun_out/exp28_r50.json 2>&1
