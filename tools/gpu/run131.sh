cd $GRAFT_REPO_ROOT
O=gpurun_out/r131; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/t.log 2>&1
echo "rc=$?" >> $O/t.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "rc=$?" >> $O/smoke.log
python bench.py > $O/b.json 2> $O/b.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/b_ref.json 2> $O/b_ref.err
python tools/cfg2_sweep.py --reps 10 --warmup 3 > $O/cfg2.log 2>&1
for c in cfg3 cfg5 cfg1; do python bench.py --no-sustained --no-cpu-baseline --steps 20 --workload $c >> $O/b_others.json 2>> $O/b.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/b_torchrun.json 2> $O/b_torchrun.err
tail -2 $O/t.log; tail -2 $O/smoke.log
