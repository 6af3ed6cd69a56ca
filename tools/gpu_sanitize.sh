#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over tools/sanitize_small.py (every kernel family)
mkdir -p gpurun_out
out=gpurun_out/sanitize.txt
: > $out
python tools/sanitize_small.py >> $out 2>&1
for tool in memcheck synccheck racecheck; do
  echo "===== $tool" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/san_$tool.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize-small|exit|Error|error" gpurun_out/san_$tool.txt | head -20 >> $out
done
