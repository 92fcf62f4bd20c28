cd $GRAFT_REPO_ROOT
PMG_CHAIN_START_GAP=1 timeout 600 python scripts/diag_chain.py 9 5 2>&1 | grep -v "batch [1-5]:" | grep -v "seg [1-9][0-9]*:" | head -30
