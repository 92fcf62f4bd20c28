# skewed-warp sweeps: parity, then the config-5 bench (one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "skew or config1 or ilut_factors" 2>&1 | tail -4
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_skew.json 2> gpurun_out/bench_skew.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_skew.err
python -c "
import json; d=json.load(open('gpurun_out/bench_skew.json'))
print('value',d['value'],'ms/step',d['ms_per_step'],'vcycle ms',d['v_cycle']['ms'], 'cycles', d['config']['cycles_per_solve'])
print({k:(round(v['ms_total'],2),v['launches']) for k,v in d['kernel_ms'].items()})"
