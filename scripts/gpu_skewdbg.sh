cd $GRAFT_REPO_ROOT
for d in ${2:-0}; do echo "== PMG_SKEW_DBG=$d"; PMG_SKEW_DBG=$d timeout 120 python scripts/diag_skew.py ${1:-9} 2>&1 | grep -E "ilut_apply|span|blk 0:|cycles"; done
