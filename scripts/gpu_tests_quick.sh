cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/dbg_wave.py 4 square 1 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bicgstab.py tests/test_cpp_api.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/quick_tests.txt
cat gpurun_out/quick_tests.txt
timeout 600 python scripts/wave_exp.py 5 9 2>&1 | tail -1
