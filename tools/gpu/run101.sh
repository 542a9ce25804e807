cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream or chained or pattern16" > gpurun_out/t101.log 2>&1
echo "rc=$?" >> gpurun_out/t101.log
python tools/host_gap.py cfg4 > gpurun_out/hg101.log 2>&1
python tools/host_gap.py cfg5 >> gpurun_out/hg101.log 2>&1
python tools/host_gap.py cfg3 >> gpurun_out/hg101.log 2>&1
SK_LIB_PATH=$PWD/paper_1708_02937_b200/libsk_rc576.so python tools/host_gap.py cfg4 >> gpurun_out/hg101.log 2>&1
SK_LIB_PATH=$PWD/paper_1708_02937_b200/libsk_rc576.so python tools/host_gap.py cfg5 >> gpurun_out/hg101.log 2>&1
python tools/host_gap.py cfg4 7500 >> gpurun_out/hg101.log 2>&1
