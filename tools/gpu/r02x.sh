cd $GRAFT_REPO_ROOT
O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_large_configs.py -m gpu -q --durations=5 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
