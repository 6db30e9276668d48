cd $GRAFT_REPO_ROOT
O=gpurun_out/r02m; mkdir -p $O
# launch list of the bench step (cold-cache, serialised), r02 code
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches.csv python bench.py --profile --steps 3 --warmup 2 --no-cpu > /dev/null 2>&1
# 8192^3 p=0.5 and cfg4 p=0.5: dX (sdd), fwd, dW, fused backward — DRAM / L2 / tensor pipe
timeout 900 ncu --set full --clock-control none -k regex:"sd_gemm" -s 6 -c 3 -o $O/t8_p05 python tools/prof_kernels.py 8192 0.5 fwd dx bwd > $O/ncu1.log 2>&1
# device timeline of back-to-back steps (SD_TRACE build)
SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so timeout 300 python tools/timeline.py 4096 0.5 3 > $O/timeline_4096.txt 2>&1
SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so timeout 300 python tools/timeline.py 1024 0.5 3 > $O/timeline_1024.txt 2>&1
