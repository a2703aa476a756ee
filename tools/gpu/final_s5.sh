# round-end validation + profiles after the FP4 window / im2col work: smoke, the whole GPU suite, the
# bench lines (ResNet-50 default, VGG-16, reference arm), the ncu launch list of the default bench command,
# and full ncu captures of the FP4 window-pair layer (ResNet-50 L1) and the im2col downsample (L13)
set -x
F=gpurun_out/r2/final5
mkdir -p $F
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $F/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $F/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $F/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $F/pytest.log
timeout 900 python bench.py > $F/bench_resnet50.log 2>&1; echo "bench rc=$?"; tail -1 $F/bench_resnet50.log | cut -c1-300
timeout 600 python bench.py --workload vgg16 > $F/bench_vgg16.log 2>&1; echo "bench vgg rc=$?"; tail -1 $F/bench_vgg16.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $F/bench_reference.log 2>&1; echo "ref rc=$?"; tail -1 $F/bench_reference.log | cut -c1-200
timeout 400 python tools/prof_layer.py --cfg 3 --layers $(seq -s, 0 51) --f4 default --opt early_weights=1 > $F/layers_r50.log 2>&1; tail -1 $F/layers_r50.log
timeout 300 python tools/prof_layer.py --cfg 4 --layers $(seq -s, 0 12) --f4 default --opt early_weights=1 > $F/layers_vgg.log 2>&1; tail -1 $F/layers_vgg.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lut_gemm|lut_conv|splitk|im2col|combine" -c 400 --csv \
   --log-file $F/launches.csv python bench.py --steps 2 --warmup 1 --no-oracle > $F/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_launches.py $F/launches.csv $F/launches.json > $F/launches.txt 2>&1; head -5 $F/launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_conv_f4 -c 1 -o $F/full_f4win_l1 \
   python tools/prof_layer.py --cfg 3 --layers 1 --f4 all --iters 1 --reps 1 > $F/ncu_win.log 2>&1; echo "ncu win rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_conv_f4 -c 1 -o $F/full_f4i2c_l13 \
   python tools/prof_layer.py --cfg 3 --layers 13 --f4 all --iters 1 --reps 1 > $F/ncu_i2c.log 2>&1; echo "ncu i2c rc=$?"
ls $F
