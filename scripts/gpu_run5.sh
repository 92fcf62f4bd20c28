cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/diag_chain.py 6 2 2>&1 | grep -E "span"
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_try12.json 2> gpurun_out/bench_try12.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_try12.err
python -c "
import json; d=json.load(open('gpurun_out/bench_try12.json'))
print('value',d['value'],'ms/step',d['ms_per_step'],'vcycle ms',d['v_cycle']['ms'])
print({k:(round(v['ms_total'],2),v['launches']) for k,v in d['kernel_ms'].items()})
print(d['roofline'])"
