cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t109.log 2>&1
echo "rc=$?" >> gpurun_out/t109.log
python tools/e2e_overlap.py cfg4 > gpurun_out/ov109.log 2>&1
python bench.py --no-sustained --no-cpu-baseline > gpurun_out/b109.json 2> gpurun_out/b109.err
python bench.py --no-sustained --no-cpu-baseline --steps 20 > gpurun_out/b109_20.json 2>> gpurun_out/b109.err
for c in cfg3 cfg5; do python bench.py --no-sustained --no-cpu-baseline --steps 20 --workload $c >> gpurun_out/b109_others.json 2>> gpurun_out/b109.err; done
