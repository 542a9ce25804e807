cd $GRAFT_REPO_ROOT
timeout 600 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream45.log 2>&1
