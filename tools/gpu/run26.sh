cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_cpp_shim.py -q -x > gpurun_out/tests26.log 2>&1
python bench.py --steps 10 --warmup 3 --no-sustained --no-cpu-baseline > gpurun_out/b26.json 2> gpurun_out/b26.err
