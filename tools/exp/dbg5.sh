for sel in "config1 and cc" "config1 and tc and not tc_ss" "config1 and tc_ss" "test_conv_vs_oracle and 1-8-8-16-16-3-1-1-0 and cc"; do
  echo "=== prior: $sel" 
  CUDA_LAUNCH_BLOCKING=1 python -m pytest tests/test_gpu_parity.py -x -q -k "($sel) or (test_conv_vs_oracle and 1-8-8-16-16-3-1-1-0 and tc and not tc_ss)" 2>&1 | grep -E "passed|failed|^E  " | head -3
done
