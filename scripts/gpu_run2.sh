cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_try2.json 2> gpurun_out/bench_try2.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_try2.err
cat gpurun_out/bench_try2.json
