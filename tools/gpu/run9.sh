cd $GRAFT_REPO_ROOT
for t in 2 4 8; do echo "== rw $t" >> gpurun_out/tile9.log; SK_LIB_PATH=variants/t$t/libsk_b200.so python tools/cfg2_sweep.py --densities 0.5,0.25,0.125 >> gpurun_out/tile9.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "cfg1 or cfg2 or layer_step or mxm or special or random_models or odd" > gpurun_out/tests9.log 2>&1
