cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15 > gpurun_out/wave_tests.txt
cat gpurun_out/wave_tests.txt
PMG_VERBOSE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/wave_bench.json 2> gpurun_out/wave_bench.err; echo "bench rc=$?"
grep -E "wave plan|rejected" gpurun_out/wave_bench.err | head -30
python - <<'PY'
import json
l=[x for x in open('gpurun_out/wave_bench.json') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print(d['ms_per_step'], d['value']); print(json.dumps(d['roofline']['per_kernel'])); print(d['kernel_ms'])
PY
