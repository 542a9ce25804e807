cd $GRAFT_REPO_ROOT
python tools/host_costs.py > gpurun_out/hc92.log 2>&1
