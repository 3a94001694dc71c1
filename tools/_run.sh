python -m paper_2506_03099_b200.build > /dev/null 2>&1
for rep in 1 2; do for ap in 0 1; do SWEEP_APPEND=$ap timeout 120 python tools/sweep.py; done; done
for rep in 1 2; do python bench.py --no-extras --no-cpu-baseline --no-e2e --stream-chunks 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'live', round(d['roofline']['achieved'],1), 'alone', round(d['roofline']['achieved_kernel_alone'],1), 'stream', round(d['streaming']['ms_per_chunk'],2))"; done
