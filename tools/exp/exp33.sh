timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp33_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp33_tests.txt
timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp33_r50.json 2>&1
DG_LIB_PATH=$PWD/bisect/lib_56152a3.so timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp33_r50_old.json 2>&1
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/exp33_r18.json 2>&1
