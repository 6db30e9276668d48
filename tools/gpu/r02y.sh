cd $GRAFT_REPO_ROOT
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_random_layers.py tests/test_dp_bench.py -m gpu -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
