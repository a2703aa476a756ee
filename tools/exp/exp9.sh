DG_LIB_PATH=$PWD/paper_2304_09049_b200/libdg_nostore.so python tools/prof_layer.py --layers 0,2,4,12 --iters 3 > gpurun_out/exp9.txt 2>&1
python tools/prof_layer.py --layers 0,2,4,12 --iters 3 >> gpurun_out/exp9.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/exp9_l0 python tools/prof_layer.py --layers 0 --iters 1 > /dev/null 2>&1
