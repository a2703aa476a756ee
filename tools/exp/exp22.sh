timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp22_tests.txt 2>&1; echo "exit $?" >> gpurun_out/exp22_tests.txt
timeout -s KILL 200 python bench.py --e2e-steps 0 --no-oracle > gpurun_out/exp22_r50.json 2>&1
DG_NO_PDL=1 timeout -s KILL 200 python bench.py --e2e-steps 0 --no-oracle > gpurun_out/exp22_r50_nopdl.json 2>&1
timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/exp22_r18.json 2>&1
DG_NO_PDL=1 timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/exp22_r18_nopdl.json 2>&1
