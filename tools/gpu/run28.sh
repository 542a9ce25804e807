cd $GRAFT_REPO_ROOT
echo "== default" > gpurun_out/tile28.log; python tools/cfg2_sweep.py --densities 0.5,0.25,0.125 >> gpurun_out/tile28.log 2>&1
for t in 04 14; do echo "== $t" >> gpurun_out/tile28.log; SK_LIB_PATH=variants/tp$t/libsk_b200.so python tools/cfg2_sweep.py --densities 0.5,0.25,0.125 >> gpurun_out/tile28.log 2>&1; done
