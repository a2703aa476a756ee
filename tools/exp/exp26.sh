timeout -s KILL 100 python tools/prof_layer.py --layers 2,4,10,12,13,25 --iters 3 > gpurun_out/exp26.txt 2>&1
echo == BN64_SHORT >> gpurun_out/exp26.txt
DG_BN64_SHORT=1 timeout -s KILL 100 python tools/prof_layer.py --layers 2,4,10,12,13,25 --iters 3 >> gpurun_out/exp26.txt 2>&1
