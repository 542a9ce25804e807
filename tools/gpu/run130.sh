cd $GRAFT_REPO_ROOT
O=gpurun_out/r130; mkdir -p $O
IS=1,2,4,8,16,32,64,128,256,512,1024,2048,4096
for b in 64 1024; do
timeout 900 python -m paper_1708_02937_b200.bench_sweep --sizes 1024,2048,4096,8192 --inverse-sparsities $IS --batch $b --repetitions 5 --warmup 2 --reference-m 1024 --output $O/sweep_b$b.csv --params $O/sweep_b${b}_params.csv > $O/sweep_b$b.log 2>&1
done
tail -3 $O/sweep_b1024.log
