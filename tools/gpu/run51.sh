cd $GRAFT_REPO_ROOT
O=gpurun_out/r51; mkdir -p $O
python tools/prof_exact.py cfg4 exact_kernel=5 exact_group=8 > $O/plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_stream -s 1 -c 1 -o $O/v3_cfg4_g8 python tools/prof_exact.py cfg4 exact_kernel=5 exact_group=8 > $O/ncu.log 2>&1
ncu -i $O/v3_cfg4_g8.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
ncu -i $O/v3_cfg4_g8.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/v3_cfg4_g8.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
