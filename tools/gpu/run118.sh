cd $GRAFT_REPO_ROOT
O=gpurun_out/r118; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
python tools/prof_dense.py 60000 2 2 > $O/eng.log 2>&1
python tools/cfg2_sweep.py --reps 5 --warmup 2 > $O/cfg2.log 2>&1
python bench.py --workload cfg1 --no-sustained --no-cpu-baseline --steps 20 > $O/b_cfg1.json 2> $O/b.err
python bench.py --no-cpu-baseline > $O/b_cfg4.json 2>> $O/b.err
tail -3 $O/t.log; cat $O/eng.log
