cd $GRAFT_REPO_ROOT
O=gpurun_out/r02small; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
