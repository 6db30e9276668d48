cd $GRAFT_REPO_ROOT
O=gpurun_out/r02zf; mkdir -p $O
for p in 0.0 0.1 0.2 0.3 0.5 0.9; do timeout 300 python tools/step_parts.py 4096 $p >> $O/parts.txt 2>&1; done
for p in 0.1 0.5; do timeout 300 python tools/step_parts.py 8192 $p 4 >> $O/parts.txt 2>&1; done
timeout 300 python tools/ab_steps.py 4096 0.1 0,1024,65536,32,64 8 >> $O/ab01.txt 2>&1
timeout 300 python tools/ab_steps.py 4096 0.2 0,1024,65536,32,64 8 >> $O/ab01.txt 2>&1
