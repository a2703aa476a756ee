# compute-sanitizer over tools/sanitize_cases.py (every kernel instance, small shapes), one tool at a time
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2/san_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/r2/san_plain.log
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-900} /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
      python tools/sanitize_cases.py ${CASES:-} > gpurun_out/r2/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -8 gpurun_out/r2/san_$tool.log
done
