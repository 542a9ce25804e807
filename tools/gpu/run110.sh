cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t110.log 2>&1
echo "rc=$?" >> gpurun_out/t110.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke110.log 2>&1
echo "rc=$?" >> gpurun_out/smoke110.log
( time python bench.py ) > gpurun_out/b110.json 2> gpurun_out/b110.err
( time python bench.py --impl reference ) > gpurun_out/b110_ref.json 2> gpurun_out/b110_ref.err
for c in cfg3 cfg5 cfg1; do python bench.py --no-sustained --no-cpu-baseline --steps 20 --workload $c >> gpurun_out/b110_others.json 2>> gpurun_out/b110.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches110.csv python bench.py --no-sustained --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu110.log 2>&1
