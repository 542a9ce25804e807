cd $GRAFT_REPO_ROOT
O=gpurun_out/r123; mkdir -p $O
for b in 15000 60000; do
timeout 900 ncu --set full --clock-control none -k regex:k_dense_engine -s 1 -c 1 -o $O/eng_b$b python tools/prof_dense.py $b 4 2 > $O/ncu_$b.log 2>&1
ncu -i $O/eng_b$b.ncu-rep --page raw --csv > $O/eng_b${b}_raw.csv 2>/dev/null
done
