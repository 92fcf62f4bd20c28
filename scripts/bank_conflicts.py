"""Shared-memory bank wavefronts of the wave kernel's value loads (diagnostics): replays the item
fill of the p=5 L factor (annulus, h = 2^-h) for a middle segment and counts, per LDS.64 of the
four term slots, the wavefronts of each half-warp (ideal 2); tries ring strides RY + delta."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
from paper_1901_01685_b200 import problems as P
from oracle import oracle as O
h=int(sys.argv[1]) if len(sys.argv)>1 else 7
pb=P.build(P.make_spec("annulus","one",(5,1),h))
A=pb.plevels[0].A
F=O.ilut_factorize(A,1e-12,1.0,O.ORDER_NONE)
L,U,perm=F.export()
n=A.nrows; seg=2**h+5
NR=32;C=4;P_=31;RY=512;DM=5
g=((n//seg)//2)|1; g0=g-1
def terms(v): return L.col[L.rowptr[v]:L.rowptr[v+1]]
cache={}
for delta in [1,2,3,4,5,6,7,8,9,12,16,17]:
  RYS=RY+delta
  tot=[]
  for t in range(60, seg - 1):
    cells=[[] for q in range(4)]
    for rl in range(32):
        base=t-P_
        s=(rl-base)%NR; ix=base+s
        if ix<0 or ix>=seg: continue
        v=g*seg+ix
        cs=terms(v); m=len(cs)
        for i,c in enumerate(cs):
            r=m-1-i
            st=0 if r<C else 1+(r-C)//C
            q=3-r if r<C else 3-(r-C)%C
            if st!=s: continue
            gc=c//seg; jx=c-gc*seg
            if gc==g and q==3 and jx==ix-s-1: continue
            cell=(DM+gc-g0)*RYS+((jx+P_)&(RY-1))
            cells[q].append((rl,cell))
    for q in range(4):
        wf=0
        for half in (0,1):
            cs=[c for (rl,c) in cells[q] if rl//16==half]
            if not cs: continue
            d={}
            for c in set(cs): d.setdefault(c%16,set()).add(c)
            wf+=max(len(x) for x in d.values())
        tot.append(wf)
  print("RYS = RY +", delta, "mean wavefronts", round(np.mean(tot),2))
