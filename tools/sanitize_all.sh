#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_run.py;
# summary lines only.  Writes gpurun_out/sanitizer.txt
out=gpurun_out/sanitizer.txt
mkdir -p gpurun_out; : > $out
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $out
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_run.py 2>&1 | grep -E "sanitize_run: done|SUMMARY|Error|error" | sort | uniq -c | head -20 >> $out
done
echo "=== initcheck (TM_TMA_EPI=0)" >> $out
TM_TMA_EPI=0 timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_run.py 2>&1 | grep -E "sanitize_run: done|SUMMARY|Uninitialized" | sort | uniq -c | head -20 >> $out
echo "=== initcheck (default TMA-store epilogue)" >> $out
timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_run.py 2>&1 | grep -E "sanitize_run: done|SUMMARY|Uninitialized.* in " | sed 's/at 0x[0-9a-f]*//' | sort | uniq -c | head -20 >> $out
