# Setup probe (one B200): config 5 assembled on the GPU + hierarchy, with the phase timers on.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/probe
PMG_VERBOSE=1 PMG_ILUT_TRACE=1 PMG_ILUT_SERIAL=${SERIAL:-0} timeout 900 python - > gpurun_out/probe/out.txt 2> gpurun_out/probe/err.txt <<'PY'
import time, sys
sys.path.insert(0, '.')
from paper_1901_01685_b200 import pmg, problems as P
t = time.time(); pb = P.build(5, assembly="gpu"); print("assembly", time.time() - t)
t = time.time(); H = pmg.build_hierarchy(pb, smoother="ilut"); print("hierarchy", time.time() - t, H.setup_seconds, H.ilut_seconds)
PY
cat gpurun_out/probe/out.txt; grep -E "setup|ilut" gpurun_out/probe/err.txt | grep -v "wave plan" | head -80
