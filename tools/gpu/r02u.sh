cd $GRAFT_REPO_ROOT
O=gpurun_out/r02u; mkdir -p $O
export SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so
ONLY=fwd,dw,dx,bwd_fused timeout 300 python tools/trace_kernels.py 4096 0.5 > $O/trace_4096.txt 2>&1
ONLY=fwd,dx,bwd_fused timeout 300 python tools/trace_kernels.py 8192 0.5 > $O/trace_8192.txt 2>&1
ONLY=fwd,dx,bwd_fused timeout 300 python tools/trace_kernels.py 4096 0.9 > $O/trace_4096_p09.txt 2>&1
