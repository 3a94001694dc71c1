# H=5 (one P=8 rank) check of the final defaults: exp split and L2 prefetch
for rep in 1 2; do
  for v in 5 1 2; do echo "poly=$v $(TM_POLY=$v SWEEP_H=5 timeout 120 python tools/sweep.py 2>&1 | tail -1)"; done
  echo "poly=5 pf=0 $(TM_L2_PREFETCH=0 SWEEP_H=5 timeout 120 python tools/sweep.py 2>&1 | tail -1)"
done > gpurun_out/ab35.txt 2>&1
timeout 600 python tools/scale_model.py gpurun_out/scale21b.json > gpurun_out/scale21b.log 2>&1
