cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -x -k "stream or exact or bench_forward" > gpurun_out/tests72.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests72.log
O=gpurun_out/r72; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
for w in cfg4 cfg3 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b72_$w.json 2>&1; done
