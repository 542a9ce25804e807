cd $GRAFT_REPO_ROOT
for v in pr64kc32cb2 pr32kc16cb2 pr64kc16cb2 pr32kc32cb1; do
  SK_LIB_PATH=$PWD/variants/lib_$v.so timeout 300 python -m pytest tests/test_gpu_scale.py -q -m gpu -x -k "cfg2" > gpurun_out/t81_$v.log 2>&1
  SK_LIB_PATH=$PWD/variants/lib_$v.so python tools/cfg2_sweep.py --densities 0.5,0.25,0.125 > gpurun_out/c81_$v.log 2>&1
done
