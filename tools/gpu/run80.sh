cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -m gpu -x -k "cfg2 or tile or mxm or layer_step" > gpurun_out/tests80.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests80.log
python tools/cfg2_sweep.py --densities 0.5,0.25,0.125,0.1 > gpurun_out/cfg2_80.log 2>&1
