python -m pytest tests -m gpu -x -q > gpurun_out/exp5_tests.txt 2>&1
echo "exit $?" >> gpurun_out/exp5_tests.txt
python tools/prof_layer.py --layers 0,1,2,4,10,11,12,13,14,16,24,25,27,28,43,44,47 --iters 3 > gpurun_out/exp5_layers.txt 2>&1
DG_NO_BRES=1 python tools/prof_layer.py --layers 0,2,4,10,12,14 --iters 3 >> gpurun_out/exp5_layers.txt 2>&1
