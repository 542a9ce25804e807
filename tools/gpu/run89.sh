cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launch89_cfg5.csv python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ncu89.log 2>&1
for i in 1 2; do python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b89_$i.json 2>&1; done
SB_BATCH=60000 python tools/step_breakdown.py cfg5 > gpurun_out/sb89.log 2>&1
