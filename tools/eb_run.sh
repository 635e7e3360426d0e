cd $GRAFT_REPO_ROOT
export SPST_DEBUG_STORE_ALL=1
timeout 600 python tools/error_budget.py --points 3 --diag 2>&1 | grep -v Warn | grep "diag\|^\[" 
timeout 600 python tools/error_budget.py --points 5 --diag 2>&1 | grep -v Warn | grep "diag\|^\["
