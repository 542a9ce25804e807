cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/tests66.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests66.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke66.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b66.json 2> gpurun_out/b66.err
python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b66_cfg3.json 2>&1
python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b66_cfg5.json 2>&1
