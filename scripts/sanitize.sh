# compute-sanitizer memcheck / synccheck / racecheck over every sweep engine.
# Logs in gpurun_out/sanitize/; copy the summaries to profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for eng in wave skew chain levels; do
  case $eng in
    wave) E="PMG_X=0";; skew) E="PMG_WAVE=0";; chain) E="PMG_WAVE=0 PMG_SKEW=0";; levels) E="PMG_FORCE_LEVELSCHED=1";;
  esac
  for tool in memcheck synccheck racecheck; do
    log=gpurun_out/sanitize/${tool}_${eng}.log
    env $E timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_driver.py > $log 2>&1
    echo "$tool $eng rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $log | tail -1)"
  done
done | tee gpurun_out/sanitize/summary.txt
head -c 1500 gpurun_out/sanitize/memcheck_wave.log
