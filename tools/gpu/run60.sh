cd $GRAFT_REPO_ROOT
for g in 1 2 4 8; do timeout 120 python tools/stream_small.py 16384 60000 246 -0.3 $g >> gpurun_out/small61.log 2>&1; done
SC_RECS=0 SC_GROUPS=0,1,2,4,8,16 timeout 600 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream61.log 2>&1
