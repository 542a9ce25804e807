cd $GRAFT_REPO_ROOT
SK_HOST_PROF=1 python tools/host_gap.py cfg4 > gpurun_out/hg100.log 2>&1
SK_HOST_PROF=1 python tools/host_gap.py cfg4 7500 >> gpurun_out/hg100.log 2>&1
python tools/host_gap.py cfg5 >> gpurun_out/hg100.log 2>&1
