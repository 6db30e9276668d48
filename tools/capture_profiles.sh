#!/usr/bin/env bash
# Run on the GPU box (via gpurun): bench line, ncu launch list of the bench
# step, one ncu --set full capture of the three GEMMs + mask kernel at the bench
# configuration. Outputs land in gpurun_out/; tools/summarize_profiles.py turns
# them into profiles/<tag>_*.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --steps 3 --warmup 2 --no-cpu > /dev/null 2>&1
# launch order per round: mask, fwd, fused backward (dW+dX); 2 warm-up rounds (+1 plan.forward) skipped
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sd_gemm|mask_plan" -s 8 -c 3 \
    -o gpurun_out/${TAG}_full python tools/prof_kernels.py 4096 0.5 mask fwd bwd > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
