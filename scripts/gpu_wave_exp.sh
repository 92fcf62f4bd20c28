cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in "" "PMG_WAVE_W=1" "PMG_WAVE=0"; do
  env $e timeout 600 python scripts/wave_exp.py 5 9 2>&1 | tail -1 | tee -a gpurun_out/wave_exp.jsonl
done
for e in "" "PMG_WAVE_W=1" "PMG_WAVE=0"; do
  env $e timeout 600 python scripts/wave_exp.py 2 10 2>&1 | tail -1 | tee -a gpurun_out/wave_exp.jsonl
done
