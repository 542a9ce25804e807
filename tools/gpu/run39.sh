cd $GRAFT_REPO_ROOT
python -m paper_1708_02937_b200.bench_sweep --sizes 512,2048 --inverse-sparsities 1,4,16,64,256,1024,4096,16384 --batch 64 --repetitions 7 --warmup 2 --seed 42 --output gpurun_out/sweep39.csv --params gpurun_out/params39.csv --reference-m 2048 > gpurun_out/sweep39.log 2>&1
