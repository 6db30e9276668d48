cd $GRAFT_REPO_ROOT
O=gpurun_out/r02l; mkdir -p $O
timeout 300 python tools/ab_settled.py 4096 0.5 "dense-default:0:dense" "dense-wide2cta:8192:dense" "cublas:0:cublas" "sparse:0:sparse" > $O/settled_4096.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"sd_gemm2" -s 4 -c 2 -o $O/ours_dense python tools/prof_kernels.py 4096 0.5 dense_nn dense_nt > $O/ncu1.log 2>&1
SD_TUNING=8192 timeout 300 ncu --set full --clock-control none -k regex:"sd_gemm2" -s 2 -c 1 -o $O/ours_dense_wide python tools/prof_kernels.py 4096 0.5 dense_nn > $O/ncu2.log 2>&1
