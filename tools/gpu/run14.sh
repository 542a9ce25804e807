cd $GRAFT_REPO_ROOT
python bench.py --workload cfg1 --steps 50 --warmup 5 --no-sustained > gpurun_out/b14_cfg1.json 2> gpurun_out/b14_cfg1.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1 or random_models or known or special or density or sparse_route" > gpurun_out/tests14.log 2>&1
python tools/prof_dense.py 60000 2 2 > gpurun_out/prof14.log 2>&1
