for rep in 1 2; do for lib in libtm.so libtm_sumguard.so; do for H in 40 5; do
 TM_LIB_PATH=$PWD/paper_2506_03099_b200/$lib SWEEP_H=$H timeout 120 python tools/sweep.py | sed "s/^/$lib /"
done; done; done
