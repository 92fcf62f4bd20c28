# Round-2 check of the setup work (one B200): ILUT parity + timing, GPU assembly parity + timing.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
timeout 1500 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -6 > gpurun_out/r2c/tests.txt
cat gpurun_out/r2c/tests.txt
PMG_VERBOSE=1 IGA_VERBOSE=1 timeout 1200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-bicgstab --time-host-assembly > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err; echo "bench rc=$?"
grep -E "^\[iga\]|\[pmg\] asm|ilut" gpurun_out/r2c/bench.err | head -60
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2c/bench.json') if l.startswith('{')][-1]); print(d['ms_per_step'], d['config'])"
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_assembly.py -x -q -m "gpu and slow" 2>&1 | tail -6 > gpurun_out/r2c/tests_slow.txt
cat gpurun_out/r2c/tests_slow.txt
