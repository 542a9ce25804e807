cd $GRAFT_REPO_ROOT
python tools/prof_dense.py 15000 2 3 > gpurun_out/prof_dense4.log 2>&1
python tools/prof_dense.py 60000 2 2 >> gpurun_out/prof_dense4.log 2>&1
python tools/cfg2_sweep.py > gpurun_out/cfg2_4.jsonl 2> gpurun_out/cfg2_4.err
timeout 900 python -m pytest tests/test_matio.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "matio or cfg1 or cfg2 or layer_step or density or mxm or special or random_models" > gpurun_out/tests4.log 2>&1
