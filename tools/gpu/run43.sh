cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/tests43.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests43.log
python bench.py --steps 10 --warmup 3 > gpurun_out/b43.json 2> gpurun_out/b43.err
python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b43_cfg5.json 2>&1
python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b43_cfg1.json 2>&1
python tools/cfg2_sweep.py > gpurun_out/cfg2_43.log 2>&1
