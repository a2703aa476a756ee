set -x
L=0,1,2,4,10,11,12,13,24,25,28,43,47
for lib in libdg libdg_noepi libdg_nost; do
  echo "== $lib"
  DG_LIB_PATH=$PWD/paper_2304_09049_b200/$lib.so python tools/prof_layer.py --layers $L --iters 3
done > gpurun_out/exp1_layers.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 2 -o gpurun_out/exp1_l1l2 python tools/prof_layer.py --layers 1,2 --iters 1 > gpurun_out/exp1_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -c 1 -o gpurun_out/exp1_l47 python tools/prof_layer.py --layers 47 --iters 1 >> gpurun_out/exp1_ncu.log 2>&1
