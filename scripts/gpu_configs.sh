# every BASELINE run (11 solves) through bench.py: time, cycles, convergence
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
run() {
  timeout 900 python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline --no-bicgstab > gpurun_out/cfg.json 2> gpurun_out/cfg.err \
    && python -c "
import json,sys; d=json.load(open('gpurun_out/cfg.json')); c=d['config']
rec={'args':'$*','workload':c['workload'],'smoother':c['smoother'],'n_dof':c['n_dof'],'ms_per_solve':d['ms_per_step'],'cycles':c['cycles_per_solve'],
     'converged':c['converged'],'final_rho':c['final_rho'],'dof_it_per_s':d['value'],'e2e':d['e2e']['value'],'sweep':d.get('triangular',{}).get('sweep_kernel'),
     'setup_s':c['setup_s']}
print(json.dumps(rec)); open('gpurun_out/configs.jsonl','a').write(json.dumps(rec)+'\n')" || echo "FAILED $*"
}
run --config 1
for p in 2 3 4; do run --config 2 --degree $p; run --config 2 --degree $p --smoother gs; done
run --config 3
run --config 4
run --config 5 --smoother gs
