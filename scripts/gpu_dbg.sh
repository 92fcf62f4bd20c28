cd $GRAFT_REPO_ROOT
timeout 300 python scripts/dbg_wave.py 4 square 1 2>&1 | tail -4
