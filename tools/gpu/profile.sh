# round profiles: launch list of the default bench command + full ncu captures of chosen kernels
mkdir -p gpurun_out/r2/prof
P=gpurun_out/r2/prof
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 2 --warmup 1 > $P/bench_plain.log 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lut_gemm|lut_conv|splitk|im2col|combine" -c 400 --csv \
   --log-file $P/launches.csv python bench.py --steps 2 --warmup 1 > $P/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_conv_f4 -c 1 -o $P/full_f4conv_l42 \
   python tools/prof_layer.py --cfg 3 --layers 42 --f4 all --iters 1 --reps 1 > $P/ncu_f4.log 2>&1; echo "ncu f4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemm_ts -c 1 -o $P/full_gemm16384 \
   python bench.py --workload gemm --n 16384 --steps 1 --warmup 0 --no-oracle > $P/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemm_ts -c 1 -o $P/full_asm_l2 \
   python tools/prof_layer.py --cfg 3 --layers 2 --iters 1 --reps 1 > $P/ncu_asm.log 2>&1; echo "ncu asm rc=$?"
ls -la $P
