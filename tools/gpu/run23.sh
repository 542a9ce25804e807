cd $GRAFT_REPO_ROOT
O=gpurun_out/r23; mkdir -p $O
# launch list of the default bench command (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
cap() {  # name regex skip cmd...
