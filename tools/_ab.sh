timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g17.log 2>&1
for rep in 1 2; do for H in 40 20 10 5; do for v in old new; do
  if [ $v = old ]; then L=paper_2506_03099_b200/libtm_old.so; else L=paper_2506_03099_b200/libtm.so; fi
  echo "$v $(TM_LIB_PATH=$L SWEEP_H=$H timeout 120 python tools/sweep.py 2>&1 | tail -1)"
done; done; done > gpurun_out/ab17.txt 2>&1
for H in 40 5; do SWEEP_H=$H timeout 200 python tools/cta_spans.py > gpurun_out/spans17_H$H.txt 2>&1; cp gpurun_out/spans_512_$H.json gpurun_out/spans17_512_$H.json; done
python -m paper_2506_03099_b200.build > /dev/null 2>&1
