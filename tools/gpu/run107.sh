cd $GRAFT_REPO_ROOT
python bench.py --no-sustained --no-cpu-baseline > gpurun_out/b107.json 2> gpurun_out/b107.err
python bench.py --no-sustained --no-cpu-baseline --steps 20 > gpurun_out/b107_20.json 2>> gpurun_out/b107.err
sed -i 's/^E2E_DEPTH = 2/E2E_DEPTH = 3/' bench.py
python bench.py --no-sustained --no-cpu-baseline --steps 20 > gpurun_out/b107_d3.json 2>> gpurun_out/b107.err
sed -i 's/^E2E_DEPTH = 3/E2E_DEPTH = 1/' bench.py
python bench.py --no-sustained --no-cpu-baseline --steps 20 > gpurun_out/b107_d1.json 2>> gpurun_out/b107.err
