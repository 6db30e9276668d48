cd $GRAFT_REPO_ROOT
O=gpurun_out/r02h; mkdir -p $O
# dense 2-CTA vs cuBLAS at 4096^3 and 8192^3, and the r02 fused backward / forward at 4096^3 p=0.5
timeout 600 ncu --set full --clock-control none -k regex:"sd_gemm|nvjet|gemm|Kernel" -s 6 -c 2 -o $O/dense_vs_cublas_4096 python tools/prof_kernels.py 4096 0.5 dense_nn cublas_nn > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"sd_gemm|nvjet|gemm|Kernel" -s 6 -c 2 -o $O/dense_vs_cublas_8192 python tools/prof_kernels.py 8192 0.5 dense_nn cublas_nn > $O/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sd_gemm|mask_plan" -s 9 -c 3 -o $O/r02_full python tools/prof_kernels.py 4096 0.5 mask fwd bwd > $O/ncu3.log 2>&1
ls -la $O
