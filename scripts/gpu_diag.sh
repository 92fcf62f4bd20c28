cd $GRAFT_REPO_ROOT
timeout 900 python scripts/diag_chain.py 9 5 2>&1 | grep -E "^.p|span|seg8|seg7"
