cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "esc or sparse_forward or thin or frontier or empty" > gpurun_out/tests35.log 2>&1
SK_ESC_DEBUG=1 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b35_dbg.json 2>&1
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b35.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_cfg3_r35.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ncu35.log 2>&1
