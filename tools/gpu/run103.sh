cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t103.log 2>&1
echo "rc=$?" >> gpurun_out/t103.log
for c in cfg4 cfg5 cfg3; do python tools/host_gap.py $c >> gpurun_out/hg103.log 2>&1; done
python tools/host_gap.py cfg4 7500 >> gpurun_out/hg103.log 2>&1
