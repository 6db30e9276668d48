cd $GRAFT_REPO_ROOT
O=gpurun_out/r02tl; mkdir -p $O
export SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so
timeout 200 python tools/timeline.py 1024 0.5 4 gate > $O/tl_1024_05.txt 2>&1
timeout 200 python tools/timeline.py 1024 0.9 4 gate > $O/tl_1024_09.txt 2>&1
