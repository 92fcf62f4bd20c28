cd $GRAFT_REPO_ROOT
for sl in 0 2 4 8; do
  PMG_WAVE_SLACK=$sl timeout 600 python scripts/wave_exp.py 5 9 2>&1 | tail -1
done
PMG_WAVE_SLACK=4 timeout 600 python scripts/diag_wave.py 9 5 2>&1 | sed -n 2,5p
PMG_WAVE_SLACK=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "skew_sweeps or gs_sweep or config1" 2>&1 | tail -2
