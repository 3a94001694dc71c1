for ic in 6 3 0; do for cfg in 512; do for H in 40 20 10 5; do
  TM_SCHED_ITEM_COST=$ic SWEEP_CFG=$cfg SWEEP_H=$H timeout 120 python tools/sweep.py | sed "s/^/ic=$ic /"
done; done; done > gpurun_out/wsk_sweep.txt 2>&1
for H in 40 5; do TM_SCHED_ITEM_COST=6 SWEEP_H=$H timeout 120 python tools/cta_spans.py | head -12; done > gpurun_out/wsk_spans.txt 2>&1
python -m paper_2506_03099_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1
tail -2 gpurun_out/pytest_gpu4.log
cat gpurun_out/wsk_sweep.txt
