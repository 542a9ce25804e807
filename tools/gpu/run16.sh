cd $GRAFT_REPO_ROOT
SK_LIB_PATH=variants/clu/libsk_b200.so python bench.py --workload cfg1 --steps 3 --warmup 3 --no-sustained --no-cpu-baseline > gpurun_out/b16.json 2> gpurun_out/b16.err
python bench.py --workload cfg1 --steps 50 --warmup 5 --no-sustained > gpurun_out/b14_cfg1.json 2> gpurun_out/b14_cfg1.err
python bench.py --workload cfg1 --steps 50 --warmup 5 --no-sustained > gpurun_out/b14_cfg1.json 2> gpurun_out/b14_cfg1.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1 or random_models or known or special or density or sparse_route" > gpurun_out/tests14.log 2>&1
