cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_bicgstab.py -x -q -m "gpu and not slow" 2>&1 | tail -15
