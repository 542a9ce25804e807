cd $GRAFT_REPO_ROOT
O=gpurun_out/r63; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
