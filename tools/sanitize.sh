for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 5 python tools/sanitize_small.py 2>&1 | grep -E "ERROR SUMMARY|sanitize driver ok|Error|error|Hazard|hazard" | head -8
done
