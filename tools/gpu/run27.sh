cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r27
( time python bench.py ) > gpurun_out/r27/bench_default.json 2> gpurun_out/r27/bench_default.err
( time python bench.py --impl reference ) > gpurun_out/r27/ref_default.json 2> gpurun_out/r27/ref_default.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r27/gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r27/smoke.log 2>&1
