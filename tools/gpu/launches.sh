mkdir -p gpurun_out/r2/prof
P=gpurun_out/r2/prof
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lut_gemm|lut_conv|splitk|im2col|combine" -c 400 --csv \
   --log-file $P/launches.csv python bench.py --steps 2 --warmup 1 > $P/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_launches.py $P/launches.csv $P/launches.json | head -12
