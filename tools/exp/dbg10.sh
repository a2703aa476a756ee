for l in 0 1 12; do echo "== vgg layer $l"; timeout -s KILL 60 python tools/prof_layer.py --cfg 4 --batch 64 --layers $l --iters 1 2>&1 | tail -2; done > gpurun_out/dbg10.txt 2>&1
for l in 0 1 12; do echo "== vgg layer $l b8"; timeout -s KILL 60 python tools/prof_layer.py --cfg 4 --batch 8 --layers $l --iters 1 2>&1 | tail -2; done >> gpurun_out/dbg10.txt 2>&1
