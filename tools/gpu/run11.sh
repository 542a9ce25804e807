cd $GRAFT_REPO_ROOT
for b in 1 4 8; do echo "== batch $b" >> gpurun_out/k1v11.log; SK_LIB_PATH=variants/b$b/libsk_b200.so python tools/cfg2_sweep.py --densities 0.1,0.01,0.001,0.0001 >> gpurun_out/k1v11.log 2>&1; done
