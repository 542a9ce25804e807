cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_cpp_shim.py -q -x -m gpu -s > gpurun_out/tests37.log 2>&1
