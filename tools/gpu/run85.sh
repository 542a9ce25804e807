cd $GRAFT_REPO_ROOT
export PE_LAYERS=3
O=gpurun_out/r85; mkdir -p $O
timeout 600 ncu --set full --sampling-interval 0 --clock-control none --import-source on -k regex:k_esc_tiny -s 1 -c 1 -o $O/tiny python tools/prof_exact.py cfg4 > $O/tiny.log 2>&1
ncu -i $O/tiny.ncu-rep --page details --csv > $O/tiny_details.csv 2>/dev/null
ncu -i $O/tiny.ncu-rep --page source --csv --print-source sass > $O/tiny_source.csv 2>/dev/null
