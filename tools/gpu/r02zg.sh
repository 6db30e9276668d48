cd $GRAFT_REPO_ROOT
O=gpurun_out/r02zg; mkdir -p $O
export SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so
for p in 0.9 0.7 0.5; do echo "## p=$p" >> $O/trace.txt; ONLY=fwd,dw,dx,bwd_fused timeout 300 python tools/trace_kernels.py 4096 $p >> $O/trace.txt 2>&1; done
timeout 300 python tools/timeline.py 4096 0.9 3 > $O/timeline09.txt 2>&1
