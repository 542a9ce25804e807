cd $GRAFT_REPO_ROOT
python tools/micro/tf32_peak.py > gpurun_out/tf32_peak.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "dense" > gpurun_out/tests21.log 2>&1
python tools/cfg2_sweep.py > gpurun_out/cfg2_21.jsonl 2> gpurun_out/cfg2_21.err
