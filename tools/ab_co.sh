#!/bin/bash
# A/B: round-1 base library vs the working tree with TM_CO_MERGE=1 (default) and =0.
for r in 1 2; do
  for v in base co1 co0; do
    case $v in
      base) lib=paper_2506_03099_b200/libtm_base.so; env="";;
      co1) lib=paper_2506_03099_b200/libtm.so; env="TM_CO_MERGE=1";;
      co0) lib=paper_2506_03099_b200/libtm.so; env="TM_CO_MERGE=0";;
    esac
    for ap in 1 0; do
      env $env TM_LIB_PATH=$lib SWEEP_APPEND=$ap SWEEP_TAG=$v SWEEP_HS=${HS:-5,10,20,40} python tools/shard_sweep.py
    done
  done
done
