cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t104.log 2>&1
echo "rc=$?" >> gpurun_out/t104.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke104.log 2>&1
python bench.py > gpurun_out/b104.json 2> gpurun_out/b104.err
for c in cfg3 cfg5 cfg1; do python bench.py --workload $c >> gpurun_out/b104_others.json 2>> gpurun_out/b104.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref104.json 2>> gpurun_out/b104.err
