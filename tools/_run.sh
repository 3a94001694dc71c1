python -m paper_2506_03099_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1
tail -2 gpurun_out/pytest_gpu6.log
for pdl in 1 0 1 0; do TM_PDL=$pdl python bench.py --no-extras --no-cpu-baseline --no-e2e --stream-chunks 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'kernel', round(d['roofline']['achieved'],1), 'stream ms/chunk', round(d['streaming']['ms_per_chunk'],2))"; done
