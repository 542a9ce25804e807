cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 2 -c 1 -o gpurun_out/tile_d025 python tools/cfg2_sweep.py --reps 2 --warmup 1 --densities 0.25 > gpurun_out/ncu10.log 2>&1
ncu -i gpurun_out/tile_d025.ncu-rep --page details --csv > gpurun_out/tile_d025_details.csv 2>/dev/null
ncu -i gpurun_out/tile_d025.ncu-rep --page raw --csv > gpurun_out/tile_d025_raw.csv 2>/dev/null
ncu -i gpurun_out/tile_d025.ncu-rep --page source --csv --print-source sass > gpurun_out/tile_d025_sass.csv 2>/dev/null
