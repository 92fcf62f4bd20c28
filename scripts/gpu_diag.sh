cd $GRAFT_REPO_ROOT
timeout 600 python scripts/diag_chain.py 9 5 2>&1 | grep -E "^.p|span|seg8 batch|prefix|seg7"
