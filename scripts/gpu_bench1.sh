cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_try.json 2> gpurun_out/bench_try.err; echo "rc=$?"
tail -5 gpurun_out/bench_try.err
cat gpurun_out/bench_try.json
