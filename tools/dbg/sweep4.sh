for ic in 3 2 1; do for wc in 0 1 2 3; do
TM_SCHED_ITEM_COST=$ic TM_SCHED_WRITE_COST=$wc SWEEP_TAG="ic=$ic wc=$wc" python tools/shard_sweep.py
done; done
