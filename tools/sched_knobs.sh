#!/bin/bash
# Schedule cost knobs (TM_SCHED_ITEM_COST / _WRITE_COST / _MERGE_COST) on the shard sweep.
for ic in ${IC:-3}; do for wc in ${WC:-0 1 2}; do for mc in ${MC:-0 1 2}; do
  TM_SCHED_ITEM_COST=$ic TM_SCHED_WRITE_COST=$wc TM_SCHED_MERGE_COST=$mc SWEEP_APPEND=${APPEND:-1} \
    SWEEP_HS=${HS:-5,10} SWEEP_TAG="ic=$ic wc=$wc mc=$mc" python tools/shard_sweep.py
done; done; done
