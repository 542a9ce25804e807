cd $GRAFT_REPO_ROOT
O=gpurun_out/r129; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "rc=$?" >> $O/smoke.log
( time python bench.py ) > $O/b.json 2> $O/b.err
( time python bench.py --impl reference ) > $O/b_ref.json 2> $O/b_ref.err
python bench.py --workload cfg3_saturated --no-cpu-baseline --no-sustained --steps 3 > $O/b_sat.json 2>> $O/b.err
tail -2 $O/t.log; tail -2 $O/smoke.log; tail -4 $O/b.err
