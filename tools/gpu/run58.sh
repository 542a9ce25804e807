cd $GRAFT_REPO_ROOT
O=gpurun_out/r58; mkdir -p $O
cap() { n=$1; shift; timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_stream -s 1 -c 1 -o $O/$n python tools/prof_exact.py "$@" > $O/$n.log 2>&1
ncu -i $O/$n.ncu-rep --page details --csv > $O/${n}_details.csv 2>/dev/null
ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
ncu -i $O/$n.ncu-rep --page source --csv --print-source sass > $O/${n}_source.csv 2>/dev/null; }
cap cfg4_g8 cfg4 exact_kernel=5 exact_group=8
cap cfg3_g1 cfg3 exact_kernel=5 exact_group=1
