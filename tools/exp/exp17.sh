L=24,26,27,28,42,43,44,45,46,47,48
timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 3 > gpurun_out/exp17.txt 2>&1
for k in 1024 2048; do echo == BN256_K $k >> gpurun_out/exp17.txt; DG_BN256_K=$k timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 3 >> gpurun_out/exp17.txt 2>&1; done
echo == BN256_K 512 no-win >> gpurun_out/exp17.txt; DG_NO_WIN=1 DG_BN256_K=512 timeout -s KILL 120 python tools/prof_layer.py --layers $L --iters 3 >> gpurun_out/exp17.txt 2>&1
