cd $GRAFT_REPO_ROOT
python tools/exact_variants.py > gpurun_out/exact_variants.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "every_variant" > gpurun_out/tests32.log 2>&1
