# Scratch command file for one gpurun call (edited per experiment):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- bash tools/eb_run.sh
# Default: the round-end checks -- smoke, the GPU parity suite, one bench line.
cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json
