#!/bin/bash
# Schedule knobs of the kept kernel on the shard sweep (zero-copy): item cost, partner-write
# cost, plain equal ranges.
for ic in 0 1 2 3 4 6 8; do
  TM_SCHED_ITEM_COST=$ic SWEEP_APPEND=0 SWEEP_HS=5,10,20 SWEEP_TAG="ic=$ic" python tools/shard_sweep.py
done
for wc in 1 2 4; do
  TM_SCHED_WRITE_COST=$wc SWEEP_APPEND=0 SWEEP_HS=5,10,20 SWEEP_TAG="ic=3 wc=$wc" python tools/shard_sweep.py
done
TM_SCHED_SPLIT=1 SWEEP_APPEND=0 SWEEP_HS=5,10,20 SWEEP_TAG="equal ranges" python tools/shard_sweep.py
