timeout 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/exp7_l0 python tools/prof_layer.py --layers 0 --iters 1 > gpurun_out/exp7_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/exp7_l2 python tools/prof_layer.py --layers 2 --iters 1 >> gpurun_out/exp7_ncu.log 2>&1
for s in 802816x64x64 802816x256x64; do python tools/trace_ts.py $s --rq; done > gpurun_out/exp7_trace.txt 2>&1
