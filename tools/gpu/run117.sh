cd $GRAFT_REPO_ROOT
O=gpurun_out/r117; mkdir -p $O
for v in b200 K L M N; do
  echo "== $v" >> $O/eng.log
  SK_LIB_PATH=$GRAFT_REPO_ROOT/paper_1708_02937_b200/libsk_$v.so timeout 300 python tools/prof_dense.py 15000 2 3 >> $O/eng.log 2>&1
  SK_LIB_PATH=$GRAFT_REPO_ROOT/paper_1708_02937_b200/libsk_$v.so timeout 300 python tools/prof_dense.py 60000 2 2 >> $O/eng.log 2>&1
done
cat $O/eng.log
