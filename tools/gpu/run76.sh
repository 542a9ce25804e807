cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/b76.json 2> gpurun_out/b76.err
python bench.py --impl reference > gpurun_out/b76_ref.json 2> gpurun_out/b76_ref.err
