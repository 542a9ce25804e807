cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/tests88.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests88.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke88.log 2>&1
for w in cfg4 cfg3 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b88_$w.json 2>&1; done
for b in 60000 7500; do SB_BATCH=$b python tools/step_breakdown.py cfg4 >> gpurun_out/sb88.log 2>&1; done
