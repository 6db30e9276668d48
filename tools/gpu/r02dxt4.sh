cd $GRAFT_REPO_ROOT
O=gpurun_out/r02dxt4; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:"sd_gemm_kernel|sd_dxt" -s 2 -c 2 -o $O/dx python tools/prof_dx.py 8192 0.5 > $O/ncu.log 2>&1
ncu -i $O/dx.ncu-rep --page raw --csv > $O/raw.csv 2>&1
rm -f $O/dx.ncu-rep
