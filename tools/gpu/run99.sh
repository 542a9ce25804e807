cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launch99_cfg3.csv python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ncu99.log 2>&1
python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b99.json 2>&1
SB_BATCH=60000 python tools/step_breakdown.py cfg3 > gpurun_out/sb99.log 2>&1
