cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_assembly.py -x -q -m "gpu and not slow" 2>&1 | tail -15 > gpurun_out/asm_tests.txt
cat gpurun_out/asm_tests.txt
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-bicgstab --time-host-assembly > gpurun_out/bench_asm.json 2> gpurun_out/bench_asm.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_asm.err
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_asm.json') if l.startswith('{')][-1]); print(d['ms_per_step'], d['config'])"
bash scripts/sanitize.sh > gpurun_out/sanitize.log 2>&1; tail -20 gpurun_out/sanitize.log
bash scripts/profile_round2.sh > gpurun_out/prof2.log 2>&1; tail -25 gpurun_out/prof2.log
