cd $GRAFT_REPO_ROOT
./scripts/ubench/step_loop3
