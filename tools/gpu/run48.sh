cd $GRAFT_REPO_ROOT
SC_RECS=0 SC_GROUPS=0,4,8,16,32 timeout 600 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream48.log 2>&1
