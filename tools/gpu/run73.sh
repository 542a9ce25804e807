cd $GRAFT_REPO_ROOT
for w in cfg4 cfg3 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b73_$1_$w.json 2>&1; done
