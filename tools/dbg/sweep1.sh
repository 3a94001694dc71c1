for rep in 1 2; do
for c in 3 2 1.5 1 0.5; do TM_SCHED_ITEM_COST=$c SWEEP_TAG="itemcost=$c" python tools/shard_sweep.py; done
done
