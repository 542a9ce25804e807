cd $GRAFT_REPO_ROOT
python tools/prof_dense.py 15000 2 3 > gpurun_out/prof_dense.log 2>&1
python tools/prof_dense.py 60000 2 2 >> gpurun_out/prof_dense.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_dense_engine -c 1 -o gpurun_out/dense_engine_sat python tools/prof_dense.py 15000 1 1 > gpurun_out/ncu_dense.log 2>&1
ncu -i gpurun_out/dense_engine_sat.ncu-rep --page details --csv > gpurun_out/dense_engine_sat_details.csv 2>/dev/null
