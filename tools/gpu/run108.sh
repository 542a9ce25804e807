cd $GRAFT_REPO_ROOT
python tools/micro/copy_interference.py > gpurun_out/ci108.log 2>&1
