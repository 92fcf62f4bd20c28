cd $GRAFT_REPO_ROOT
for v in "" NO_STG NO_RHS NO_RESET NO_XBSEL CHK4; do
  if [ -z "$v" ]; then E=""; else E="PMG_CUDA_LIB=libpmg_cuda_$v.so"; fi
  echo "== $v $(env $E timeout 300 python scripts/diag_wave.py 9 5 2>&1 | grep -E 'blk 0|same CTA' | tr '\n' ' ')"
done
