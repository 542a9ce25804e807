cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_cpp_shim.py tests/test_gpu_parity.py -q -m gpu -k "shim or acceptance or dense" > gpurun_out/tests38.log 2>&1
./tests/cpp/_ref/acceptance > gpurun_out/acceptance38.log 2>&1
