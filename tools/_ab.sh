# same-lib A/B of the next-item Q prefetch: TM_Q_PREFETCH = loads before the item end (0 = off)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/g32.log 2>&1
for rep in 1 2 3; do for v in 0 8 16; do
  TM_Q_PREFETCH=$v python bench.py --no-extras --no-cpu-baseline --no-e2e --stream-chunks 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('qpf=$v', round(d['value'],1), 'live', round(r['achieved'],1), 'alone', round(r['achieved_kernel_alone'],1), 'chunk1', round(d['chunk1']['tflops_per_gpu'],1), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab32.txt 2>&1
for rep in 1 2; do for cfg in "512 40" "512 5"; do set -- $cfg; for v in 0 8; do
  echo "qpf=$v $(TM_Q_PREFETCH=$v SWEEP_CFG=$1 SWEEP_H=$2 timeout 120 python tools/sweep.py 2>&1 | tail -1)"
  echo "qpf=$v $(TM_Q_PREFETCH=$v SWEEP_CFG=$1 SWEEP_H=$2 SWEEP_APPEND=1 timeout 120 python tools/sweep.py 2>&1 | tail -1)"
done; done; done >> gpurun_out/ab32.txt 2>&1
