cd $GRAFT_REPO_ROOT
O=gpurun_out/r93; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg5_bench.csv python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch5.log 2>&1
python bench.py > gpurun_out/b93.json 2> gpurun_out/b93.err
for w in cfg3 cfg5 cfg1; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b93_$w.json 2>&1; done
