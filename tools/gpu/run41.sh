cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_cpp_shim.py -q -m gpu > gpurun_out/tests41.log 2>&1
./tests/cpp/_ref/acceptance > gpurun_out/acceptance41.log 2>&1
python -m paper_1708_02937_b200.bench_sweep --sizes 512,2048 --inverse-sparsities 1,4,16,64,256,1024,4096,16384 --batch 64 --repetitions 7 --warmup 2 --seed 42 --output gpurun_out/sweep41.csv --params gpurun_out/params41.csv --reference-m 2048 > gpurun_out/sweep41.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep41.csv python -m paper_1708_02937_b200.bench_sweep --sizes 512,2048 --inverse-sparsities 1,4,16384 --batch 64 --repetitions 3 --warmup 1 --seed 42 --output gpurun_out/sweep41n.csv > /dev/null 2>&1
