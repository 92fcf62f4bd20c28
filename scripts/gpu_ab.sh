# A/B of an alternative build of the CUDA library (PMG_CUDA_LIB=<file in lib/>): parity tests of the
# sweeps, then the default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
for lib in "$@"; do
  echo "== $lib"
  PMG_CUDA_LIB=$lib timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -2
  PMG_CUDA_LIB=$lib PMG_VERBOSE=1 timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-bicgstab > gpurun_out/ab/$lib.json 2> gpurun_out/ab/$lib.err; echo "rc=$?"
  grep "wave plan n=10" gpurun_out/ab/$lib.err | head -4
  python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/ab/$lib.json') if l.startswith('{')][-1])
print('$lib', 'ms/solve %.2f' % d['ms_per_step'], {k: round(v['ms'],3) for k,v in d['roofline']['per_kernel'].items()}, 'coarse', round(d['kernel_ms']['coarse']['ms_total'],2), d['config']['final_rho'])
PY
done
