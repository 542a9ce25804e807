cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "cfg1 or cfg2 or layer_step or mxm or special or random_models or odd" > gpurun_out/tests7.log 2>&1
python tools/cfg2_sweep.py > gpurun_out/cfg2_7.jsonl 2> gpurun_out/cfg2_7.err
