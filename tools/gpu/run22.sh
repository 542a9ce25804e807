cd $GRAFT_REPO_ROOT
O=gpurun_out/r22; mkdir -p $O
# launch list of the default bench command (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/launches_cfg4_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu_launch.log 2>&1
cap() {  # name regex skip cmd...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o $O/$name "$@" > $O/$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
}
cap exact_cfg4 k_exact_layer 3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap exact_cfg5 k_exact_layer 3 python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap exact_cfg3 k_exact_layer 3 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
cap tile_cfg2_d05 k_spmm_tile 2 python tools/cfg2_sweep.py --reps 1 --warmup 2 --densities 0.5
cap gemm_cfg2 k_gemm_packed 2 python tools/cfg2_sweep.py --reps 1 --warmup 2 --densities 0.5
cap engine_sat k_dense_engine 1 python tools/prof_dense.py 15000 1 1
cap cluster_cfg1 k_dense_cluster 3 python bench.py --workload cfg1 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained
