cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dense_cluster -s 3 -c 1 -o gpurun_out/cluster_cfg1 python bench.py --workload cfg1 --steps 2 --warmup 3 --no-sustained --no-cpu-baseline > gpurun_out/ncu13.log 2>&1
ncu -i gpurun_out/cluster_cfg1.ncu-rep --page details --csv > gpurun_out/cluster_cfg1_details.csv 2>/dev/null
ncu -i gpurun_out/cluster_cfg1.ncu-rep --page raw --csv > gpurun_out/cluster_cfg1_raw.csv 2>/dev/null
