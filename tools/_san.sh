for L in old new; do
  if [ $L = old ]; then export TM_LIB_PATH=paper_2506_03099_b200/libtm_old.so; else export TM_LIB_PATH=paper_2506_03099_b200/libtm.so; fi
  echo "=== $L"; timeout 600 compute-sanitizer --tool initcheck --print-limit 6 python tools/sanitize_run.py 2>&1 | head -60
done > gpurun_out/san19.txt 2>&1
