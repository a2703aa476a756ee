for L in bisect/lib_56152a3.so paper_2304_09049_b200/libdg.so; do
DG_LIB_PATH=$PWD/$L timeout -s KILL 200 python bench.py --steps 30 > gpurun_out/exp31.json 2>&1
echo $L $(tail -1 gpurun_out/exp31.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('gemm_ms_per_layer'))") >> gpurun_out/exp31.txt
done
