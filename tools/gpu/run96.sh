cd $GRAFT_REPO_ROOT
SK_HOST_PROF=1 SB_BATCH=7500 python tools/step_breakdown.py cfg4 > gpurun_out/hp96.log 2>&1
SK_HOST_PROF=1 SB_BATCH=60000 python tools/step_breakdown.py cfg4 >> gpurun_out/hp96.log 2>&1
