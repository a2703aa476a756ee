python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or conv or prepared or config1" > gpurun_out/exp2_tests.txt 2>&1
echo "exit $?" >> gpurun_out/exp2_tests.txt
python tools/prof_layer.py --layers 0,1,2,4,10,11,12,13,24,25,28,43,47 --iters 3 > gpurun_out/exp2_layers.txt 2>&1
