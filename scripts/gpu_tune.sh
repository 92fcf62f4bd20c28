cd $GRAFT_REPO_ROOT
for cfg in "64 64" "48 64" "32 64" "64 32" "80 48"; do
  set -- $cfg
  echo "AHEAD=$1 GAP=$2: $(PMG_CHAIN_AHEAD=$1 PMG_CHAIN_START_GAP=$2 timeout 300 python scripts/diag_chain.py 9 5 2>&1 | grep -E 'span' | sed 's/per-seg fin duration median [0-9.]* us;//; s/fin_start lag median [0-9.]* us//' | tr '\n' ' ')"
done
