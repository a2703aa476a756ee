for lib in libdg_noepi libdg_skel; do echo "== $lib"; DG_LIB_PATH=$PWD/paper_2304_09049_b200/$lib.so python tools/prof_layer.py --layers 0,2,4,12 --iters 3 2>&1; done > gpurun_out/exp10.txt
for lib in libdg_skel; do echo "== UNP4 $lib"; DG_TS_UNP4=1 DG_LIB_PATH=$PWD/paper_2304_09049_b200/$lib.so python tools/prof_layer.py --layers 0,2,4,12 --iters 3 2>&1; done >> gpurun_out/exp10.txt
