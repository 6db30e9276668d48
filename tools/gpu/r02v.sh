cd $GRAFT_REPO_ROOT
O=gpurun_out/r02v; mkdir -p $O
export SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so
SD_TUNING=80 ONLY=dense_nn,dense_nt,dense_tn,fwd,dx timeout 300 python tools/trace_kernels.py 4096 0.5 > $O/trace_dense1cta_narrow.txt 2>&1
SD_TUNING=48 ONLY=dense_nn,dense_nt,dense_tn,fwd,dx timeout 300 python tools/trace_kernels.py 4096 0.5 > $O/trace_dense1cta_wide.txt 2>&1
