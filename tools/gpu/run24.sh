cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke24.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "exact or scale or sparse or esc or frontier or density or column or layer_on" > gpurun_out/tests24.log 2>&1
for c in cfg4 cfg3 cfg5; do python bench.py --workload $c --steps 10 --warmup 3 --no-sustained --no-cpu-baseline > gpurun_out/b24_$c.json 2> gpurun_out/b24_$c.err; done
