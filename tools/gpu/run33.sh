cd $GRAFT_REPO_ROOT
python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b33.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ncu33.log 2>&1
