cd $GRAFT_REPO_ROOT
O=gpurun_out/r119; mkdir -p $O
python tools/prof_dense.py 60000 2 2 > $O/eng.log 2>&1
python tools/prof_dense.py 15000 2 3 >> $O/eng.log 2>&1
python tools/cfg2_sweep.py --reps 10 --warmup 3 > $O/cfg2.log 2>&1
cat $O/eng.log
