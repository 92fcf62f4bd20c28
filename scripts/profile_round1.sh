# Round-1 evidence: plain bench, ncu launch list of the timed region, ncu --set full of the
# top kernels.  Run under gpurun (1 GPU).  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
PMG_PROFILE_REGION=1 $B > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
PMG_PROFILE_REGION=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
PMG_PROFILE_REGION=1 timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name-base function -k regex:"^k_skew$|^k_chain$|^k_rowop$" -c 6 -o gpurun_out/prof_full $B > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ls -la gpurun_out | tail -8
