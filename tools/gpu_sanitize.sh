# compute-sanitizer passes over tools/sanitize_step.py (outputs gpurun_out/r2_sanitizer_*.txt)
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_step.py > gpurun_out/r2_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2_sanitizer_$tool.txt
done
