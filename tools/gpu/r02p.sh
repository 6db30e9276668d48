cd $GRAFT_REPO_ROOT
O=gpurun_out/r02p; mkdir -p $O
timeout 600 python tools/ab_libs.py paper_2411_01238_b200/lib/libsparsedrop_b200.so tools/ablibs/lib_before.so 8192 0.5 8 > $O/ab_8192_p05_rev.txt 2>&1
timeout 400 python tools/ab_libs.py paper_2411_01238_b200/lib/libsparsedrop_b200.so tools/ablibs/lib_before.so 4096 0.5 12 > $O/ab_4096_p05_rev.txt 2>&1
timeout 400 python tools/ab_libs.py tools/ablibs/lib_before.so paper_2411_01238_b200/lib/libsparsedrop_b200.so 65536,8192,8192 0.5 3 > $O/ab_cfg4_p05.txt 2>&1
