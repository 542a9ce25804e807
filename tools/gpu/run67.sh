cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/tests67.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests67.log
