cd $GRAFT_REPO_ROOT
O=gpurun_out/r69; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pad_passes -s 1 -c 1 -o $O/pad python tools/prof_exact.py cfg4 > $O/pad.log 2>&1
ncu -i $O/pad.ncu-rep --page details --csv > $O/pad_details.csv 2>/dev/null
ncu -i $O/pad.ncu-rep --page source --csv --print-source sass > $O/pad_source.csv 2>/dev/null
