cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -x -k "esc or bench_forward or thin or smoke" > gpurun_out/tests84.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests84.log
export PE_LAYERS=3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_esc_tiny" -c 3 --csv --log-file gpurun_out/esc84.csv python tools/prof_exact.py cfg4 > gpurun_out/esc84.log 2>&1
unset PE_LAYERS
python tools/step_breakdown.py cfg4 > gpurun_out/sb84.log 2>&1
for w in cfg4; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/b84_$w.json 2>&1; done
