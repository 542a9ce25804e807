cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/tests17.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench17.json 2> gpurun_out/bench17.err
