cd $GRAFT_REPO_ROOT
for b in 1 2 4 8; do
  echo "== batch $b" >> gpurun_out/variants6.log
  SK_LIB_PATH=variants/b$b/libsk_b200.so python tools/prof_dense.py 60000 2 2 >> gpurun_out/variants6.log 2>&1
  SK_LIB_PATH=variants/b$b/libsk_b200.so python tools/prof_dense.py 15000 2 3 >> gpurun_out/variants6.log 2>&1
done
