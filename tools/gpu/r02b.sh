# round-2 GPU check: full gpu suite (incl. large configs), racecheck after the
# scheduler-lane fix, short bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
for tune in 0 384; do
  SD_TUNING=$tune timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_steps.py --steps 96 > $O/san_racecheck_$tune.txt 2>&1; echo "rc=$?" >> $O/san_racecheck_$tune.txt
done
SD_TUNING=0 timeout 300 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_steps.py --steps 512 > $O/san_synccheck_512.txt 2>&1; echo "rc=$?" >> $O/san_synccheck_512.txt
SD_TUNING=0 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_steps.py --steps 1024 > $O/san_memcheck_1024.txt 2>&1; echo "rc=$?" >> $O/san_memcheck_1024.txt
timeout 600 python bench.py --no-e2e --no-cpu > $O/bench.json 2> $O/bench.err
