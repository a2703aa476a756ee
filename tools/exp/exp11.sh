./tools/sync_bench > gpurun_out/exp11.txt 2>&1; ./tools/sync_bench_hint >> gpurun_out/exp11.txt 2>&1
for lib in libdg libdg_hint; do echo "== $lib"; DG_LIB_PATH=$PWD/paper_2304_09049_b200/$lib.so python tools/prof_layer.py --layers 0,2,12,27,28,47 --iters 3 2>&1; done >> gpurun_out/exp11.txt
