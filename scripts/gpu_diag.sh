cd $GRAFT_REPO_ROOT
timeout 600 python scripts/diag_chain.py ${1:-10} ${2:-5} 2>&1 | tail -60
