# quick timing of the square GEMM (bench gemm workload) under option settings
mkdir -p gpurun_out/r2
for o in ${OPTS:-"tma_store=1"}; do
  echo "=== $o"
  DG_OPTS="$o" timeout 300 python bench.py --workload gemm --n ${N:-16384} --steps 10 --warmup 3 --no-oracle 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['value'], d['compute_only'], d['roofline']['frac_vs_i8_mma_ceiling'], d['config']['kernel'])
    else: print(l.rstrip()[:300])"
done 2>&1 | tee gpurun_out/r2/${TAG}_gemm.log
