for L in base pub; do echo "== $L"; TPF_LIB_PATH=_ab/$L.so python tools/trace_virtual.py 8 cfg2 steady; done > gpurun_out/tr_steady.txt 2>&1
