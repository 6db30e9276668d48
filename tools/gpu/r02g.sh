cd $GRAFT_REPO_ROOT
O=gpurun_out/r02g; mkdir -p $O
timeout 300 python tools/ab_graph.py 4096 0.5 8 > $O/ab_graph_4096.txt 2>&1
timeout 300 python tools/ab_graph.py 1024 0.5 8 > $O/ab_graph_1024.txt 2>&1
timeout 400 python tools/ab_graph.py 8192 0.5 4 > $O/ab_graph_8192.txt 2>&1
