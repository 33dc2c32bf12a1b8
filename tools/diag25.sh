python tools/sanitize_new_paths.py > gpurun_out/san_plain.log 2>&1; tail -1 gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_new_paths.py > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" gpurun_out/san_$tool.log | head -8
done
