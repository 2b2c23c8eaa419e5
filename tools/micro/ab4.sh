python tools/ab_up.py _ab/prev/libtpfuse_b200.so _ab/p1/libtpfuse_b200.so 2
python tools/ab_up.py _ab/p2/libtpfuse_b200.so _ab/d2p1/libtpfuse_b200.so 2
python tools/ab_up.py _ab/d2p2/libtpfuse_b200.so _ab/prev/libtpfuse_b200.so 2
