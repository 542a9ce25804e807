cd $GRAFT_REPO_ROOT
O=gpurun_out/r98; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:k_exact_tma -s 1 -c 1 -o $O/tma_cfg4 python tools/prof_exact.py cfg4 exact_kernel=6 exact_group=8 > $O/tma.log 2>&1
ncu -i $O/tma_cfg4.ncu-rep --page details --csv > $O/tma_details.csv 2>/dev/null
ncu -i $O/tma_cfg4.ncu-rep --page raw --csv > $O/tma_raw.csv 2>/dev/null
