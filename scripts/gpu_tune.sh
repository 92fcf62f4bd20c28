cd $GRAFT_REPO_ROOT
for c in 48 32 20; do
  PMG_CHAIN_GAP_CAP=$c timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err
  python -c "
import json; d=json.load(open('gpurun_out/t.json'))
print('CAP $c ms/step',round(d['ms_per_step'],1),{k:round(v['ms_total']/max(v['launches'],1),2) for k,v in d['kernel_ms'].items() if v['launches']})"
done
