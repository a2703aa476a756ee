for L in bisect/lib_56152a3.so paper_2304_09049_b200/libdg.so; do
n=$(basename $L .so)
for layer in 1; do
DG_LIB_PATH=$PWD/$L timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:lut_gemm_ts -s 1 -c 1 -o gpurun_out/exp34_${n}_$layer python tools/prof_layer.py --layers $layer --iters 2 > gpurun_out/exp34_ncu_$n.log 2>&1
done
done
