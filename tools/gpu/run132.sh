cd $GRAFT_REPO_ROOT
O=gpurun_out/r132; mkdir -p $O; rm -f $O/eng.log
for v in A B C D E F G; do
  echo "== $v" >> $O/eng.log
  SK_LIB_PATH=$GRAFT_REPO_ROOT/paper_1708_02937_b200/libsk_$v.so timeout 300 python tools/prof_dense.py 60000 6 2 >> $O/eng.log 2>&1
  SK_LIB_PATH=$GRAFT_REPO_ROOT/paper_1708_02937_b200/libsk_$v.so timeout 300 python tools/prof_dense.py 7500 6 3 >> $O/eng.log 2>&1
done
cat $O/eng.log
