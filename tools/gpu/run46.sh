cd $GRAFT_REPO_ROOT
O=gpurun_out/r46; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_stream -s 2 -c 1 -o $O/stream_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sustained > $O/ncu.log 2>&1
ncu -i $O/stream_cfg4.ncu-rep --page details --csv > $O/stream_cfg4_details.csv 2>/dev/null
ncu -i $O/stream_cfg4.ncu-rep --page raw --csv > $O/stream_cfg4_raw.csv 2>/dev/null
ncu -i $O/stream_cfg4.ncu-rep --page source --csv --print-source sass > $O/stream_cfg4_source.csv 2>/dev/null
