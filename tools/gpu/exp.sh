# time layers with experimental library variants (DG_LIB_PATH) against the product library
mkdir -p gpurun_out/r2
for v in ${VARIANTS:-libdg}; do
  echo "=== $v"
  DG_LIB_PATH=$PWD/paper_2304_09049_b200/$v.so timeout 300 python tools/prof_layer.py $PROF 2>&1 | grep -v identical
done > gpurun_out/r2/${TAG}_exp.log 2>&1
cat gpurun_out/r2/${TAG}_exp.log
