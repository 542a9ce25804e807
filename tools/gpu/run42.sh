cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/tests42.log 2>&1
./tests/cpp/_ref/acceptance > gpurun_out/acceptance42.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/b42.json 2> gpurun_out/b42.err
