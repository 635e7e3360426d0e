cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench_gramfill2.json 2> gpurun_out/bench_gramfill2.err; tail -c 400 gpurun_out/bench_gramfill2.json
