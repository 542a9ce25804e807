cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r19
python bench.py --steps 10 --warmup 3 > gpurun_out/r19/bench_cfg4.json 2> gpurun_out/r19/bench_cfg4.err
python bench.py --workload cfg3 --steps 10 --warmup 3 --no-sustained > gpurun_out/r19/bench_cfg3.json 2> gpurun_out/r19/bench_cfg3.err
python bench.py --workload cfg5 --steps 10 --warmup 3 --no-sustained > gpurun_out/r19/bench_cfg5.json 2> gpurun_out/r19/bench_cfg5.err
python bench.py --workload cfg1 --steps 50 --warmup 5 > gpurun_out/r19/bench_cfg1.json 2> gpurun_out/r19/bench_cfg1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r19/ref_cfg4.json 2> gpurun_out/r19/ref_cfg4.err
python tools/cfg2_sweep.py > gpurun_out/r19/cfg2.jsonl 2> gpurun_out/r19/cfg2.err
