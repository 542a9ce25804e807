cd $GRAFT_REPO_ROOT
python bench.py --workload cfg1 --steps 50 --warmup 5 --no-sustained > gpurun_out/b12_cfg1.json 2> gpurun_out/b12_cfg1.err
python tools/prof_dense.py 60000 2 2 > gpurun_out/prof12.log 2>&1
python tools/prof_dense.py 15000 2 3 >> gpurun_out/prof12.log 2>&1
python tools/cfg2_sweep.py > gpurun_out/cfg2_12.jsonl 2> gpurun_out/cfg2_12.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests12.log 2>&1
