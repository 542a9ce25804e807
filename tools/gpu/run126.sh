cd $GRAFT_REPO_ROOT
O=gpurun_out/r126; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
python tools/cfg2_sweep.py --reps 10 --warmup 3 > $O/cfg2.log 2>&1
python bench.py --no-cpu-baseline > $O/b_cfg4.json 2> $O/b.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_engine -s 1 -c 1 -o $O/engine_staged_b60000 python tools/prof_dense.py 60000 3 2 > $O/ncu.log 2>&1
ncu -i $O/engine_staged_b60000.ncu-rep --page raw --csv > $O/engine_staged_raw.csv 2>/dev/null
ncu -i $O/engine_staged_b60000.ncu-rep --page details --csv > $O/engine_staged_details.csv 2>/dev/null
tail -3 $O/t.log
