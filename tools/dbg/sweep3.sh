for rep in 1 2; do
SWEEP_TAG="base" python tools/shard_sweep.py
TM_DBG_NOMERGE=1 SWEEP_TAG="nomerge" python tools/shard_sweep.py
TM_SCHED_ITEM_COST=0 SWEEP_TAG="cost0" python tools/shard_sweep.py
TM_DBG_NOMERGE=1 TM_SCHED_ITEM_COST=0 SWEEP_TAG="nomerge cost0" python tools/shard_sweep.py
done
