cd $GRAFT_REPO_ROOT
O=gpurun_out/r02large; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_random_layers.py -q -k large --durations=10 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
