cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:k_esc_sample -c 2 -o gpurun_out/esc_sample python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-sustained > gpurun_out/ncu36.log 2>&1
