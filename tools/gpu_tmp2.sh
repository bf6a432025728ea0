L=paper_1604_05937_b200/_native/libprismesh_cuda.so
for v in notrow trow; do cp build/exp/$v.so $L; python tools/dbg_p2.py gpurun_out/y_$v.npy 5; done
