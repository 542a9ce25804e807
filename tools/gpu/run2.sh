cd $GRAFT_REPO_ROOT
python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python bench.py --workload cfg5 --shard cols --steps 5 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/bench_cols.json 2> gpurun_out/bench_cols.err
MASTER_ADDR=127.0.0.1 MASTER_PORT=29511 RANK=0 LOCAL_RANK=0 WORLD_SIZE=1 python tools/colshard_timing.py cfg5 > gpurun_out/colshard.log 2>&1
python bench.py --workload cfg1 --steps 20 --warmup 5 --no-sustained > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
python tools/cfg2_sweep.py > gpurun_out/cfg2.jsonl 2> gpurun_out/cfg2.err
