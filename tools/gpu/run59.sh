cd $GRAFT_REPO_ROOT
SK_DEBUG_STREAM=1 timeout 120 python tools/stream_small.py 262144 60000 262 -0.45 16 > gpurun_out/small59.log 2>&1
