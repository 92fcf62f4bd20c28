cd $GRAFT_REPO_ROOT
timeout 120 python -c "
import numpy as np, time
from paper_1901_01685_b200 import pmg, problems as P
from oracle import oracle as O
pb=P.build(1)
A=pb.plevels[1].A
t=time.time(); F=pmg.ilut_factorize(A,1e-12,1.0,'none'); print('fact',time.time()-t, F.stats(), flush=True)
r=np.random.default_rng(0).uniform(-1,1,A.nrows)
t=time.time(); e=pmg.ilut_apply(F,r); print('apply', time.time()-t, flush=True)
Fo=O.ilut_factorize(A,1e-12,1.0,O.ORDER_NONE)
print('bitwise', np.array_equal(e.view(np.uint64), Fo.apply(r).view(np.uint64)))
"; echo "rc=$?"
