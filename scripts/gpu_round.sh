cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_round.json
