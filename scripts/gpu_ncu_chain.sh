cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PMG_CHAIN_GATE_DIST=3
timeout 300 python scripts/diag_chain.py 9 5 > gpurun_out/diag_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:^k_chain$ -s 2 -c 1 -o gpurun_out/chain_prof4 python scripts/diag_chain.py 9 5 > gpurun_out/ncu_chain.log 2>&1; echo "ncu rc=$?"
