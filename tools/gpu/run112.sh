cd $GRAFT_REPO_ROOT
O=gpurun_out/r112; mkdir -p $O
for c in cfg3 cfg5; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_$c.csv python bench.py --workload $c --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_$c.log 2>&1
done
python tools/step_breakdown.py cfg3 > $O/steps_cfg3.log 2>&1
