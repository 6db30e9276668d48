cd $GRAFT_REPO_ROOT
O=gpurun_out/r03g; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sd_gemm" -s 2 -c 2 \
    -o $O/bwd python tools/prof_kernels.py 4096 0.5 bwd dense_nt > $O/ncu.log 2>&1
ncu -i $O/bwd.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/bwd.ncu-rep --page raw --csv > $O/raw.csv 2>&1
rm -f $O/bwd.ncu-rep
