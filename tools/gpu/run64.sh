cd $GRAFT_REPO_ROOT
for g in 1 2 4 8; do timeout 120 python tools/stream_small.py 4096 3000 1000 -0.1 $g 4 >> gpurun_out/small64.log 2>&1; done
for g in 1 2 4 8; do timeout 120 python tools/stream_small.py 16384 60000 246 -0.3 $g 4 >> gpurun_out/small64.log 2>&1; done
SC_FIELDS=4,8 SC_GROUPS=0,2,4,8 timeout 900 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream64.log 2>&1
