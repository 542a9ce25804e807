cd $GRAFT_REPO_ROOT
SC_KERNEL=6 SC_FIELDS=0 SC_GROUPS=0,4,8,16 timeout 900 python tools/stream_check.py cfg4 cfg3 cfg5 > gpurun_out/stream97.log 2>&1
