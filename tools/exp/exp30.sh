timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp30_a.json 2>&1
DG_NO_SPLITK=1 timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp30_b.json 2>&1
timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp30_c.json 2>&1
DG_NO_SPLITK=1 timeout -s KILL 200 python bench.py --workload resnet18 --steps 200 > gpurun_out/exp30_d.json 2>&1
