cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -s 2>&1 | grep -v Warn | tail -12
