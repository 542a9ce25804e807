cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "staged or column or publish or row_block" > gpurun_out/tests25.log 2>&1
python bench.py --workload cfg5 --shard cols --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b25_cols.json 2> gpurun_out/b25_cols.err
