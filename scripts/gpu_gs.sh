# GS smoother timing: skewed-warp vs chained sweeps (config 2, p = 4; config 5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sk in 1 0; do
  for c in "--config 2 --degree 4" "--config 5"; do
    PMG_SKEW=$sk timeout 900 python bench.py $c --smoother gs --steps 1 --warmup 1 --no-cpu-baseline --no-bicgstab > gpurun_out/gs_$sk.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/gs_$sk.json'))
print('PMG_SKEW=$sk', '$c', 'ms/step', round(d['ms_per_step'],2), 'cycles', d['config']['cycles_per_solve'], 'conv', d['config']['converged'], 'gs_fine ms', round(d['kernel_ms']['gs_fine']['ms_total'],2), d['kernel_ms']['gs_fine']['launches'])"
  done
done
