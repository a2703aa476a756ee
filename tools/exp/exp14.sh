timeout -s KILL 100 python tools/prof_layer.py --layers 2,3,12,13,25,26,44 --iters 3 > gpurun_out/exp14.txt 2>&1
echo == BN256S >> gpurun_out/exp14.txt
DG_TS_BN256S=1 timeout -s KILL 100 python tools/prof_layer.py --layers 2,3,12,13,25,26,44 --iters 3 >> gpurun_out/exp14.txt 2>&1
