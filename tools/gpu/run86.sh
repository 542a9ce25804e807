cd $GRAFT_REPO_ROOT
for w in cfg4 cfg3 cfg5; do
  SK_LIB_PATH=$PWD/variants/lib_mb20.so python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b86_mb20_$w.json 2>&1
done
SK_LIB_PATH=$PWD/variants/lib_mb20.so timeout 600 python -m pytest tests/test_gpu_scale.py -q -m gpu -x -k "bench_forward" > gpurun_out/t86.log 2>&1
