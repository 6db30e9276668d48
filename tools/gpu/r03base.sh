cd $GRAFT_REPO_ROOT
O=gpurun_out/r03base; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
