cd $GRAFT_REPO_ROOT
O=gpurun_out/r125; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
python tools/cfg2_sweep.py --reps 10 --warmup 3 > $O/cfg2.log 2>&1
tail -3 $O/t.log
