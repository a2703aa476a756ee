python -m pytest tests -m gpu -x -q > gpurun_out/exp8_tests.txt 2>&1
echo "exit $?" >> gpurun_out/exp8_tests.txt
python tools/prof_layer.py --layers 0,1,2,4,10,11,12,13,14,16,24,25,27,28,43,44,47 --iters 3 > gpurun_out/exp8_layers.txt 2>&1
echo == UNP4 >> gpurun_out/exp8_layers.txt
DG_TS_UNP4=1 python tools/prof_layer.py --layers 0,4,5 --iters 3 >> gpurun_out/exp8_layers.txt 2>&1
