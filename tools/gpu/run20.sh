cd $GRAFT_REPO_ROOT
python bench.py --workload cfg5 --shard cols --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b20_cols.json 2> gpurun_out/b20_cols.err
MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 RANK=0 LOCAL_RANK=0 WORLD_SIZE=1 python bench.py --workload cfg5 --shard cols --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b20_cols_dist.json 2> gpurun_out/b20_cols_dist.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "column or publish or row_block" > gpurun_out/tests20.log 2>&1
