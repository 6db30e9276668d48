cd $GRAFT_REPO_ROOT
O=gpurun_out/r02gs; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernel_modes.py -m gpu -q -x -k "graph" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python tools/isolated_probe.py > $O/iso.jsonl 2> $O/iso.err
