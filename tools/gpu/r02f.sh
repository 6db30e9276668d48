cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernel_modes.py tests/test_gpu_comm.py -m gpu -q -x > $O/pytest_modes.txt 2>&1; echo "rc=$?" >> $O/pytest_modes.txt
timeout 600 python bench.py --no-e2e --no-cpu > $O/bench_graph.json 2> $O/bench_graph.err
timeout 600 python bench.py --no-e2e --no-cpu --no-graph --no-sweep > $O/bench_eager.json 2> $O/bench_eager.err
