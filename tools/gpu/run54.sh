cd $GRAFT_REPO_ROOT
for g in 4 8 16 32; do timeout 120 python tools/stream_small.py 65536 60000 262 -0.35 $g >> gpurun_out/small54.log 2>&1; done
for g in 4 8 16 32; do timeout 120 python tools/stream_small.py 16384 60000 246 -0.3 $g >> gpurun_out/small54.log 2>&1; done
for g in 4 8 16 32; do timeout 120 python tools/stream_small.py 262144 60000 262 -0.45 $g >> gpurun_out/small54.log 2>&1; done
SC_RECS=0 SC_GROUPS=0,4,8,16,32 timeout 600 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream54.log 2>&1
