#!/bin/bash
# Re-run the default bench N times (reduced streaming/e2e/cpu) and report failures.
N=${1:-5}
for i in $(seq 1 $N); do
  timeout 900 python bench.py --no-cpu-baseline --stream-chunks 8 > gpurun_out/stress_$i.json 2> gpurun_out/stress_$i.err
  rc=$?
  echo "run $i rc=$rc $(grep -m1 -o 'File .*bench.py", line [0-9]*, in [a-z_]*' gpurun_out/stress_$i.err | tail -1) $(grep -m1 -o 'CUDA error: [a-z ]*' gpurun_out/stress_$i.err)"
done
