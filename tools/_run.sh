python -m paper_2506_03099_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1
tail -2 gpurun_out/pytest_gpu5.log
for rep in 1 2; do for H in 40 5; do SWEEP_H=$H timeout 120 python tools/sweep.py; done; SWEEP_CFG=720 timeout 120 python tools/sweep.py; done
