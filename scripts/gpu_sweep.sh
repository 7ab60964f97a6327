for tool in memcheck racecheck synccheck; do
  for path in 1 2; do
    echo "== $tool path $path"
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py $path 2>&1 | grep -E "ERROR SUMMARY|path|Error|error" | head -8
  done
done
