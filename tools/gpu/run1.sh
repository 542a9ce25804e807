cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/scale.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_scale.py > gpurun_out/gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
