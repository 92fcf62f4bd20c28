cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in "" "PMG_CUDA_LIB=libpmg_cuda_chk4.so"; do
  echo "== $lib" | tee -a gpurun_out/diag_wave2.txt
  env $lib timeout 600 python scripts/diag_wave.py 9 5 2>&1 | head -5 | tee -a gpurun_out/diag_wave2.txt
  env $lib timeout 600 python scripts/wave_exp.py 5 9 2>&1 | tail -1 | tee -a gpurun_out/diag_wave2.txt
done
