cd $GRAFT_REPO_ROOT
O=gpurun_out/r02dp; mkdir -p $O
timeout 900 python -m pytest tests/test_dp_bench.py tests/test_gpu_comm.py -m gpu -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e > $O/cfg5.json 2> $O/cfg5.err; echo "rc=$?" >> $O/cfg5.err
