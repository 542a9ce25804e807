cd $GRAFT_REPO_ROOT
export PE_LAYERS=3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_esc_tiny|k_pad|k_gather|k_rp_from|Scan" -c 80 --csv --log-file gpurun_out/esc83.csv python tools/prof_exact.py cfg4 > gpurun_out/esc83.log 2>&1
