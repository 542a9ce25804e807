cd $GRAFT_REPO_ROOT
python tools/step_breakdown.py cfg4 > gpurun_out/sb77.log 2>&1
