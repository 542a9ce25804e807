cd $GRAFT_REPO_ROOT
timeout 300 compute-sanitizer --print-limit 5 python tools/stream_small.py 4096 3000 60 -0.2 > gpurun_out/san53.log 2>&1
timeout 300 python tools/stream_small.py 65536 60000 262 -0.35 > gpurun_out/small53.log 2>&1
