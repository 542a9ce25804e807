cd $GRAFT_REPO_ROOT
O=gpurun_out/r120; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wide_batch or cfg1 or random_models or sparse_route or density_switch" > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
timeout 120 python tools/prof_dense.py 60000 2 2 > $O/eng.log 2>&1
timeout 120 python tools/prof_dense.py 15000 2 3 >> $O/eng.log 2>&1
tail -5 $O/t.log; cat $O/eng.log
