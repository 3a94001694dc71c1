# exp split A/B: TM_POLY=1 (all MUFU, default) vs 5 (1/16 polynomial), full bench minus extras/e2e/cpu
for rep in 1 2 3; do for v in 1 5; do
  TM_POLY=$v python bench.py --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('poly=$v', round(d['value'],1), 'live', round(r['achieved'],1), 'alone', round(r['achieved_kernel_alone'],1), 'chunk1', round(d['chunk1']['tflops_per_gpu'],1), 'stream_ms', round(d['streaming']['ms_per_chunk'],2), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab34.txt 2>&1
