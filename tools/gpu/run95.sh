cd $GRAFT_REPO_ROOT
O=gpurun_out/r95; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pad -s 1 -c 1 -o $O/pad5 python tools/prof_exact.py cfg5 > $O/pad5.log 2>&1
ncu -i $O/pad5.ncu-rep --page details --csv > $O/pad5_details.csv 2>/dev/null
ncu -i $O/pad5.ncu-rep --page raw --csv > $O/pad5_raw.csv 2>/dev/null
ncu -i $O/pad5.ncu-rep --page source --csv --print-source sass > $O/pad5_source.csv 2>/dev/null
