cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/diag_chain.py 8 5 > gpurun_out/diag_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_chain -s 2 -c 1 -o gpurun_out/chain_prof3 python scripts/diag_chain.py 8 5 > gpurun_out/ncu_chain.log 2>&1; echo "ncu rc=$?"
