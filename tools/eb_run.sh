cd $GRAFT_REPO_ROOT
timeout 120 ./build/tma_il_probe
