for rep in 1 2; do
TM_EXIT_WAIT_FULL=1 SWEEP_TAG="exit_full" python tools/shard_sweep.py
SWEEP_TAG="exit_read" python tools/shard_sweep.py
done
