# bench step A/B of the L2 prefetch depth: TM_L2_PREFETCH = K/V tiles of the first item (0 = off)
for rep in 1 2 3; do for v in 0 2 4 8; do
  TM_L2_PREFETCH=$v python bench.py --no-extras --no-cpu-baseline --no-e2e --stream-chunks 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('pf=$v', round(d['value'],1), 'live', round(r['achieved'],1), 'alone', round(r['achieved_kernel_alone'],1), 'chunk1', round(d['chunk1']['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab29.txt 2>&1
