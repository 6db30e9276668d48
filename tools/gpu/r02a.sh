set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02a/pytest_gpu.txt
for t in memcheck synccheck racecheck; do
  for tune in 0 384; do
    SD_TUNING=$tune timeout 300 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_steps.py --steps 96 > gpurun_out/r02a/san_${t}_${tune}.txt 2>&1
    echo "rc=$?" >> gpurun_out/r02a/san_${t}_${tune}.txt
  done
done
SD_TUNING=0 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_steps.py --steps 1024 > gpurun_out/r02a/san_memcheck_1024.txt 2>&1; echo "rc=$?" >> gpurun_out/r02a/san_memcheck_1024.txt
tail -3 gpurun_out/r02a/*.txt
