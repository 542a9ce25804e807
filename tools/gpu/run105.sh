cd $GRAFT_REPO_ROOT
python tools/e2e_timeline.py 6 > gpurun_out/tl105.log 2>&1
python tools/host_gap.py cfg4 > gpurun_out/hg105.log 2>&1
python tools/step_breakdown.py > gpurun_out/sb105.log 2>&1
