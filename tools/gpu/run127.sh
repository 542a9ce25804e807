cd $GRAFT_REPO_ROOT
O=gpurun_out/r127; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "wide or staged or density_switch or cfg1 or random_models or sparse_route or cfg2" > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
for b in 60000 7500; do timeout 200 python tools/prof_dense.py $b 6 2 >> $O/eng.log 2>&1; done
tail -3 $O/t.log; cat $O/eng.log
