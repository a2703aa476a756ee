mkdir -p gpurun_out/s4
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/s4/full_l1 python tools/prof_layer.py --layers 1 --iters 1 > gpurun_out/s4/ncu_l1.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/s4/full_l2 python tools/prof_layer.py --layers 2 --iters 1 > gpurun_out/s4/ncu_l2.log 2>&1
