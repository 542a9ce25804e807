cd $GRAFT_REPO_ROOT
O=gpurun_out/r111; mkdir -p $O
# the driver's N>1 launch form at world size 1 (NCCL init, barrier, max-over-ranks path)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-sustained --no-cpu-baseline > $O/b_torchrun.json 2> $O/b_torchrun.err
echo "rc=$?" >> $O/b_torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 1 --steps 5 --warmup 3 --no-sustained --no-cpu-baseline --workload cfg5 --shard cols > $O/b_cols.json 2> $O/b_cols.err
echo "rc=$?" >> $O/b_cols.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 1 --steps 5 --warmup 3 --no-sustained --no-cpu-baseline --workload cfg5 --shard cols --exchange peer > $O/b_cols_peer.json 2> $O/b_cols_peer.err
echo "rc=$?" >> $O/b_cols_peer.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29520 bench.py --impl reference --gpus 1 --steps 1 --warmup 0 > $O/b_ref_torchrun.json 2> $O/b_ref_torchrun.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
cap() {  # name regex skip cmd...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o $O/$name "$@" > $O/$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
}
cap stream_cfg4 k_exact_stream 3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap stream_cfg5 k_exact_stream 3 python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
