cd $GRAFT_REPO_ROOT
python tools/e2e_timeline.py 6 > gpurun_out/tl91.log 2>&1
