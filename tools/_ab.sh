# bench step A/B of the tail schedule: TM_SCHED_LEAD=0 (previous) vs 1 (default), interleaved
for rep in 1 2 3; do for v in 0 1; do
  TM_SCHED_LEAD=$v python bench.py --no-extras --no-cpu-baseline --no-e2e --stream-chunks 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('lead=$v', round(d['value'],1), 'live', round(r['achieved'],1), 'alone', round(r['achieved_kernel_alone'],1), 'chunk1', round(d['chunk1']['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab26.txt 2>&1
