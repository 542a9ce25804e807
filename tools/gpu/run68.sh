cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "stream or exact" > gpurun_out/tests68.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests68.log
O=gpurun_out/r68; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b68.json 2> gpurun_out/b68.err
