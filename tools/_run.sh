python -m paper_2506_03099_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu12.log 2>&1
tail -1 gpurun_out/pytest_gpu12.log
python bench.py > gpurun_out/bench_v10.json 2> gpurun_out/bench_v10.err
python bench.py --config wan720 --no-extras > gpurun_out/bench_v10_720.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v10_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-extras --stream-chunks 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fmha_sm100 -s 14 -c 1 -o gpurun_out/v10_full_append -f python bench.py --steps 4 --warmup 3 --no-e2e --no-extras --stream-chunks 0 --no-cpu-baseline > /dev/null 2>&1
SWEEP_H=5 ncu --set full --clock-control none --import-source on -k regex:fmha_sm100 -s 30 -c 1 -o gpurun_out/v10_full_h5 -f python tools/sweep.py > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
