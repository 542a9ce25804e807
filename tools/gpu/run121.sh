cd $GRAFT_REPO_ROOT
O=gpurun_out/r121; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wide_batch or cfg1 or random_models or sparse_route or density_switch" > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
for b in 15000 30000 60000; do timeout 200 python tools/prof_dense.py $b 6 2 >> $O/eng.log 2>&1; done
tail -5 $O/t.log; cat $O/eng.log
