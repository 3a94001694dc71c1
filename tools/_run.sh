python -m paper_2506_03099_b200.build > /dev/null 2>&1
TM_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --stream-chunks 2 > gpurun_out/bench2proc.log 2>&1
echo rc=$?
tail -c 400 gpurun_out/bench2proc.log
