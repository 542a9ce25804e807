cd $GRAFT_REPO_ROOT
O=gpurun_out/r113; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exact_stream -s 28 -c 1 -o $O/stream_cfg4_banked python tools/bank_layout.py cfg4 > $O/ncu.log 2>&1
ncu -i $O/stream_cfg4_banked.ncu-rep --page raw --csv > $O/stream_cfg4_banked_raw.csv 2>/dev/null
ncu -i $O/stream_cfg4_banked.ncu-rep --page details --csv > $O/stream_cfg4_banked_details.csv 2>/dev/null
