cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "chained" > gpurun_out/tests90.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests90.log
