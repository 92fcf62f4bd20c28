# ncu --set full of the rotating-lane sweeps inside the timed region of the default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-bicgstab"
PMG_PROFILE_REGION=1 timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name-base function -k regex:"^k_wave$" -c 4 -o gpurun_out/wave_full $B > gpurun_out/ncu_wave.log 2>&1; echo "full rc=$?"
tail -5 gpurun_out/ncu_wave.log
