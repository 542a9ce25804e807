cd $GRAFT_REPO_ROOT
SK_DEBUG_STREAM=1 timeout 120 python tools/stream_small.py 65536 60000 262 -0.35 8 > gpurun_out/small56.log 2>&1
