# Round-2 evidence run (one B200): GPU tests, the default bench line, every BASELINE run as a
# bench line with its CPU baseline.  Outputs in gpurun_out/r2/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2/gpu_tests.txt
cat gpurun_out/r2/gpu_tests.txt
timeout 1200 python bench.py --steps 5 --warmup 3 --cpu-single-thread --time-host-assembly > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err; echo "default rc=$?"
run() {
  name=$1; shift
  timeout 900 python bench.py "$@" --steps 3 --warmup 3 --no-bicgstab > gpurun_out/r2/cfg_$name.json 2> gpurun_out/r2/cfg_$name.err; echo "$name rc=$?"
}
run c1 --config 1
for p in 2 3 4; do run c2p${p}_ilut --config 2 --degree $p; run c2p${p}_gs --config 2 --degree $p --smoother gs; done
run c3 --config 3
run c4 --config 4
run c5_gs --config 5 --smoother gs
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2/*.json')):
    try:
        d = json.loads([l for l in open(f) if l.startswith('{')][-1])
    except Exception as e:
        print(f, 'no line', e); continue
    c = d['config']; cb = d.get('cpu_baseline') or {}
    print(f.split('/')[-1], c['workload'], c['smoother'], 'ms/solve %.2f' % d['ms_per_step'], 'cycles', c['cycles_per_solve'],
          'conv', c['converged'], 'value %.3g' % d['value'], 'cpu %.3g' % (cb.get('value') or 0), 'launches', d['gpu_launches'])
PY
