cd $GRAFT_REPO_ROOT
python tools/e2e_overlap.py cfg4 > gpurun_out/ov106.log 2>&1
