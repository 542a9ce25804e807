cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream or chained or pattern16" > gpurun_out/t102.log 2>&1
echo "rc=$?" >> gpurun_out/t102.log
for c in cfg4 cfg5 cfg3; do python tools/host_gap.py $c >> gpurun_out/hg102.log 2>&1; done
python tools/host_gap.py cfg5 0 exact_layout=2 >> gpurun_out/hg102.log 2>&1
python tools/host_gap.py cfg4 0 exact_layout=1 >> gpurun_out/hg102.log 2>&1
for c in cfg4 cfg5; do SK_LIB_PATH=$PWD/paper_1708_02937_b200/libsk_rc512.so python tools/host_gap.py $c >> gpurun_out/hg102.log 2>&1; done
