cd $GRAFT_REPO_ROOT
O=gpurun_out/r03h; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q > $O/pytest.txt 2>&1
timeout 300 python tools/e2e_slots.py 4096 0.5 > $O/e2e.txt 2>&1
timeout 900 python tools/fig4_bench.py --sizes 1024,2048,4096 --out $O/fig4.csv > $O/fig4.log 2>&1
