#!/bin/bash
# A/B of two in-tree builds on the shard sweep (one rank's heads at P = 2/4/8 and P = 1):
#   tools/ab_shard.sh <libA.so> <libB.so> [reps]
A=$1; B=$2; N=${3:-2}
for r in $(seq 1 $N); do
  for lib in $A $B; do
    for ap in 1 0; do
      TM_LIB_PATH=$lib SWEEP_APPEND=$ap SWEEP_TAG=$(basename $lib) python tools/shard_sweep.py
    done
  done
done
