#!/bin/bash
O=gpurun_out/${1:-r02san}
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --target-processes all python tools/sanitize_run.py > $O/$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|workload done|Error|error" $O/$tool.txt | head -5 >> $O/summary.txt
done
cat $O/summary.txt
