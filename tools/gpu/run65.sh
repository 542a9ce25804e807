cd $GRAFT_REPO_ROOT
timeout 120 python tools/stream_small.py 65536 4096 2000 -0.1 4 4 >> gpurun_out/small65.log 2>&1
timeout 120 python tools/stream_small.py 65536 4096 2000 -0.1 8 4 >> gpurun_out/small65.log 2>&1
timeout 120 python tools/stream_small.py 16384 60000 246 -0.3 1 4 >> gpurun_out/small65.log 2>&1
SC_FIELDS=0 SC_GROUPS=0,8,16 timeout 900 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream65.log 2>&1
