cd $GRAFT_REPO_ROOT
O=gpurun_out/r02san2; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck python tools/sanitize_steps.py --steps 256 > $O/san_memcheck.txt 2>&1
timeout 900 $CS --tool synccheck python tools/sanitize_steps.py --steps 96 > $O/san_synccheck.txt 2>&1
timeout 1200 $CS --tool racecheck python tools/sanitize_steps.py --steps 96 > $O/san_racecheck.txt 2>&1
for f in $O/san_*.txt; do echo "$f: $(grep -h 'sanitize_steps ok' $f | tail -1) | $(grep -h 'SUMMARY' $f | tail -1)"; done > $O/summary.txt
