cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "esc or sparse_forward or thin or frontier or empty" > gpurun_out/tests34.log 2>&1
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b34.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_cfg3_r34.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ncu34.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b34_cfg4.json 2>&1
