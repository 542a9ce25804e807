cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke18.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x > gpurun_out/tests18.log 2>&1
python bench.py --steps 10 --warmup 3 --no-sustained --no-cpu-baseline > gpurun_out/b18_cfg4.json 2> gpurun_out/b18_cfg4.err
python bench.py --workload cfg3 --steps 10 --warmup 3 --no-sustained --no-cpu-baseline > gpurun_out/b18_cfg3.json 2> gpurun_out/b18_cfg3.err
