cd $GRAFT_REPO_ROOT
for b in 60000 15000 7500; do SB_BATCH=$b python tools/step_breakdown.py cfg4 >> gpurun_out/sb87.log 2>&1; done
