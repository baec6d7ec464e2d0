# compute-sanitizer over scripts/sanitize_target.py; summaries -> gpurun_out/san_*.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_target.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.log
  tail -3 gpurun_out/san_$tool.log >> gpurun_out/san_summary.log
done
