cd $GRAFT_REPO_ROOT
O=gpurun_out/r122; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 200 > $O/smi.log 2>&1 &
SMI=$!
sleep 1; echo "--- B=15000 L=24" >> $O/smi.log
timeout 200 python tools/prof_dense.py 15000 24 3 > $O/eng.log 2>&1
echo "--- B=60000 L=6" >> $O/smi.log
timeout 200 python tools/prof_dense.py 60000 6 3 >> $O/eng.log 2>&1
kill $SMI
cat $O/eng.log
