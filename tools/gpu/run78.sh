cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -x -k "stream or exact or bench_forward" > gpurun_out/tests78.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests78.log
for w in cfg4 cfg3 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b78_$w.json 2>&1; done
