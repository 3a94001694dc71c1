for rep in 1 2; do for lib in libtm.so libtm_lsu.so; do TM_LIB_PATH=$PWD/paper_2506_03099_b200/$lib SWEEP_APPEND=1 timeout 120 python tools/sweep.py | sed "s/^/$lib /"; done; done
TM_LIB_PATH=$PWD/paper_2506_03099_b200/libtm_lsu.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "zero_copy or layers or ragged or wan512 or few_units" 2>&1 | tail -2
