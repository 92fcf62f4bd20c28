# Final check of a round (one B200): the whole GPU suite, smoke(), the default bench line, then the
# profile script.  Outputs in gpurun_out/final/ and gpurun_out/prof2/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -6 > gpurun_out/final/gpu_tests.txt; cat gpurun_out/final/gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/final/smoke.txt
timeout 1200 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "reference rc=$?"
tail -c 600 gpurun_out/final/bench_default.json; echo; tail -c 400 gpurun_out/final/bench_reference.json
bash scripts/profile_round2.sh > gpurun_out/prof2.log 2>&1; tail -12 gpurun_out/prof2.log
