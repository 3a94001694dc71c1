python -m paper_2506_03099_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.log 2>&1
tail -2 gpurun_out/pytest_gpu11.log
for rep in 1 2; do for H in 40 20 10 5; do SWEEP_H=$H timeout 120 python tools/sweep.py; done; SWEEP_CFG=720 timeout 120 python tools/sweep.py; SWEEP_CFG=720 SWEEP_H=5 timeout 120 python tools/sweep.py; done
python bench.py --no-extras --no-cpu-baseline --stream-chunks 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'live', round(d['roofline']['achieved'],1), 'alone', round(d['roofline']['achieved_kernel_alone'],1), 'e2e', round(d['e2e']['value'],1), 'stream', round(d['streaming']['ms_per_chunk'],2))"
