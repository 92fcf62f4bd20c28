# full GPU test suite + default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/check_tests.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; echo "bench rc=$?"
cat gpurun_out/check_tests.txt
python - <<'PY'
import json
l=[x for x in open('gpurun_out/check_bench.json') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print('ms/step', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'], 'launches', d['gpu_launches'])
    print({k:round(v['ms'],3) for k,v in d['roofline']['per_kernel'].items()}); print({k:(round(v['ms_total'],2),v['launches']) for k,v in d['kernel_ms'].items()})
    print('cpu', (d.get('cpu_baseline') or {}).get('value'))
PY
tail -3 gpurun_out/check_bench.err
