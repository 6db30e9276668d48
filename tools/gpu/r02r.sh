cd $GRAFT_REPO_ROOT
O=gpurun_out/r02r; mkdir -p $O
timeout 600 python tools/ab_libs.py tools/ablibs/lib_b.so tools/ablibs/lib_c.so 8192 0.5 8 > $O/ab_8192_p05.txt 2>&1
timeout 400 python tools/ab_libs.py tools/ablibs/lib_c.so tools/ablibs/lib_b.so 4096 0.5 12 > $O/ab_4096_p05.txt 2>&1
timeout 400 python tools/ab_libs.py tools/ablibs/lib_b.so tools/ablibs/lib_c.so 4096 0.9 12 > $O/ab_4096_p09.txt 2>&1
timeout 400 python tools/ab_libs.py tools/ablibs/lib_c.so tools/ablibs/lib_b.so 65536,8192,8192 0.5 3 > $O/ab_cfg4_p05.txt 2>&1
