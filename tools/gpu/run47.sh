cd $GRAFT_REPO_ROOT
SC_RECS=0 timeout 600 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream47.log 2>&1
