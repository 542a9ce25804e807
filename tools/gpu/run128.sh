cd $GRAFT_REPO_ROOT
O=gpurun_out/r128; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_engine -s 1 -c 1 -o $O/engine_staged_b60000 python tools/prof_dense.py 60000 3 2 > $O/ncu.log 2>&1
ncu -i $O/engine_staged_b60000.ncu-rep --page raw --csv > $O/engine_staged_raw.csv 2>/dev/null
ncu -i $O/engine_staged_b60000.ncu-rep --page details --csv > $O/engine_staged_details.csv 2>/dev/null
