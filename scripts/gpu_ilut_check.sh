# ILUT parity (factors bitwise vs the oracle) + setup probe in both scheduling modes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/probe
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" -k "ilut or factor or solve or bitwise" 2>&1 | tail -4
for mode in 0 1; do
PMG_VERBOSE=1 PMG_ILUT_TRACE=1 PMG_ILUT_SERIAL=$mode timeout 900 python - > gpurun_out/probe/out_$mode.txt 2> gpurun_out/probe/err_$mode.txt <<'PY'
import time, sys
sys.path.insert(0, '.')
from paper_1901_01685_b200 import pmg, problems as P
t = time.time(); pb = P.build(5, assembly="gpu"); print("assembly", time.time() - t)
t = time.time(); H = pmg.build_hierarchy(pb, smoother="ilut"); print("hierarchy", time.time() - t, H.setup_seconds, H.ilut_seconds)
PY
echo "serial=$mode"; cat gpurun_out/probe/out_$mode.txt; grep -E "ilut trace|ilut n=" gpurun_out/probe/err_$mode.txt | head -12
done
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -m "gpu and slow" 2>&1 | tail -3
