cd $GRAFT_REPO_ROOT
O=gpurun_out/r75; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
cap() {  # name regex skip cmd...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o $O/$name "$@" > $O/$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
}
cap stream_cfg4 k_exact_stream 3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap stream_cfg5 k_exact_stream 3 python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap stream_cfg3 k_exact_stream 3 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap pad_cfg4 k_pad_passes 3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
