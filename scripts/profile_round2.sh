# Round-2 evidence (one B200): plain bench line under the profile region, ncu launch list of the
# timed region, ncu --set full of the hot kernels (ILUT solve: fine L/U sweeps, p=1 sweeps, SpMV
# family, dense coarse solve; GS solve: GS sweep + upper-sum pre-pass; GPU ILUT factorization on
# config 3; GPU assembly on config 3).  The reports are exported to CSV on the box (raw page,
# demangled names) and deleted -- gpurun brings back at most 64 MiB; only the small source-level
# capture of the two fine sweeps is kept as .ncu-rep.  Outputs in gpurun_out/prof2/; summarised by
# scripts/summarize_profiles.py.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-bicgstab"
export_csv() {  # $1 = report without extension
  ncu -i $1.ncu-rep --page raw --csv --print-kernel-base demangled > $1_raw.csv 2> $1_export.err && rm -f $1.ncu-rep
}
PMG_PROFILE_REGION=1 $B > $O/prof_plain.json 2> $O/prof_plain.err; echo "plain rc=$?"
PMG_PROFILE_REGION=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv $B > $O/ncu_launches.log 2>&1; echo "launch list rc=$?"
PMG_PROFILE_REGION=1 timeout 2400 ncu --profile-from-start off --set full --clock-control none \
    --kernel-name-base function -k regex:"^k_wave$|^k_rowop$|^k_dense_solve$|^k_wave_upd$" -c 36 -o $O/prof_full $B > $O/ncu_full.log 2>&1; echo "full rc=$?"
export_csv $O/prof_full
PMG_PROFILE_REGION=1 timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name-base function -k regex:"^k_wave$" -c 2 -o $O/fine_sweeps_source $B > $O/ncu_src.log 2>&1; echo "source rc=$?"
ncu -i $O/fine_sweeps_source.ncu-rep --page raw --csv --print-kernel-base demangled > $O/fine_sweeps_source_raw.csv 2>/dev/null
PMG_PROFILE_REGION=1 timeout 1500 ncu --profile-from-start off --set full --clock-control none \
    --kernel-name-base function -k regex:"^k_wave$|^k_wave_gs_su$" -c 3 -o $O/gs_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-bicgstab --smoother gs > $O/ncu_gs.log 2>&1; echo "gs rc=$?"
export_csv $O/gs_full
timeout 1500 ncu --set full --clock-control none --kernel-name-base function -k regex:"^k_ilut$|^k_asm_elements$|^k_asm_gather$|^k_asm_rowsum$" -c 40 \
    -o $O/setup_full python -c "
import sys; sys.path.insert(0, '.')
from paper_1901_01685_b200 import pmg, problems as P
pb = P.build(3, assembly='gpu')
F = pmg.ilut_factorize(pb.plevels[0].A, 1e-12, 1.0, 'none')
print(F.stats())" > $O/ncu_setup.log 2>&1; echo "setup rc=$?"
export_csv $O/setup_full
du -sh $O; ls -la $O
