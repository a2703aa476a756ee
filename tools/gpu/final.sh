# round-end validation: build + smoke, the whole GPU suite, the bench lines (ResNet-50 default, VGG-16,
# reference arm) and the ncu launch list of the default bench command
set -x
mkdir -p gpurun_out/r2/final
F=gpurun_out/r2/final
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $F/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $F/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $F/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $F/pytest.log
timeout 900 python bench.py > $F/bench_resnet50.log 2>&1; echo "bench rc=$?"; tail -1 $F/bench_resnet50.log | cut -c1-400
timeout 600 python bench.py --workload vgg16 > $F/bench_vgg16.log 2>&1; echo "bench vgg rc=$?"; tail -1 $F/bench_vgg16.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $F/bench_reference.log 2>&1; echo "ref rc=$?"; tail -1 $F/bench_reference.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lut_gemm|lut_conv|splitk|im2col|combine" -c 400 --csv \
   --log-file $F/launches.csv python bench.py --steps 2 --warmup 1 --no-oracle > $F/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_launches.py $F/launches.csv $F/launches.json > $F/launches.txt 2>&1; head -5 $F/launches.txt
