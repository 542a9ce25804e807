cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 0 -c 1 -o gpurun_out/tile_d05 python tools/cfg2_sweep.py --reps 2 --warmup 1 --densities 0.5 > gpurun_out/ncu8a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 0 -c 1 -o gpurun_out/tile_d01 python tools/cfg2_sweep.py --reps 2 --warmup 1 --densities 0.1 > gpurun_out/ncu8b.log 2>&1
for r in tile_d05 tile_d01; do ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null; done
