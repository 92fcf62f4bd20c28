cd $GRAFT_REPO_ROOT
for d in 2 3; do
echo "DIST$d: $(PMG_CHAIN_GATE_DIST=$d timeout 600 python scripts/diag_chain.py 9 5 2>&1 | grep -E 'sweep span' | sed 's/fin_start lag median [0-9.]* us//' | tr '\n' ' ' | cut -c1-300)"
done
echo "SERIAL: $(PMG_CHAIN_START_GAP=100000 timeout 600 python scripts/diag_chain.py 9 5 2>&1 | grep -E 'sweep span' | head -1 | sed 's/fin_start lag median [0-9.]* us//' | tr '\n' ' ' | cut -c1-300)"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
