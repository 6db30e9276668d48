cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
for tune in 0 384; do
  SD_TUNING=$tune timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_steps.py --steps 96 > $O/san_racecheck_$tune.txt 2>&1; echo "rc=$?" >> $O/san_racecheck_$tune.txt
done
