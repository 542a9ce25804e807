cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_cpp_shim.py -q -x -k "cfg2 or mxm or layer_step or dense or shim or random" > gpurun_out/tests29.log 2>&1
python tools/cfg2_sweep.py > gpurun_out/cfg2_29.jsonl 2> gpurun_out/cfg2_29.err
