cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -x -k "stream or exact or bench_forward or chained" > gpurun_out/tests94.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests94.log
O=gpurun_out/r94; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pad -c 4 --csv --log-file $O/pad.csv python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-sustained > $O/ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pad -c 4 --csv --log-file $O/pad4.csv python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-sustained > $O/ncu4.log 2>&1
for w in cfg4 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b94_$w.json 2>&1; done
