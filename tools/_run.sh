python -m paper_2506_03099_b200.build > /dev/null 2>&1
python bench.py > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v8_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-extras --stream-chunks 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fmha_sm100 -s 30 -c 1 -o gpurun_out/v8_full -f python tools/sweep.py > gpurun_out/v8_ncu.log 2>&1
SWEEP_H=5 ncu --set full --clock-control none --import-source on -k regex:fmha_sm100 -s 30 -c 1 -o gpurun_out/v8_full_h5 -f python tools/sweep.py > gpurun_out/v8_ncu_h5.log 2>&1
TM_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --stream-chunks 2 > gpurun_out/bench2proc_e2e.log 2>&1
echo rc=$?
tail -c 600 gpurun_out/bench_v8.json
