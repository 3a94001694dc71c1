python -m paper_2506_03099_b200.build > /dev/null 2>&1
python bench.py > gpurun_out/bench_v9b.json 2> gpurun_out/bench_v9b.err
ncu --set full --clock-control none --import-source on -k regex:fmha_sm100 -s 14 -c 1 -o gpurun_out/v9_full_append -f python bench.py --steps 4 --warmup 3 --no-e2e --no-extras --stream-chunks 0 --no-cpu-baseline > gpurun_out/v9_ncu_append.log 2>&1
