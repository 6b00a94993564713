"""Fraction of a view's tiles touched by the pruned rows of each pruning level
(C3, CPU, oracle projection): the upper bound on what dirty-tile reuse across
levels could skip -- with UNIFORM RANDOM usage, which the real
sweep does not have (its measured clean shares: DESIGN.md s4, level sweep).
python tools/dirty_tiles.py"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import airgs_oracle as orc
from paper_2512_20943_b200 import synth
cfg=synth.CONFIGS['C3']
seq=synth.Sequence(cfg, seed=0, event_every=0)
gt0=seq.frame(0); gt1=seq.frame(1)
cams=synth.cameras(cfg)
cam=cams[0]
n=gt0.shape[0]
rng=np.random.default_rng(1)
diff=np.abs(gt1-gt0).max(axis=1)>1e-9
idx=np.nonzero(diff)[0]
print("delta rows",idx.size)
usage=rng.integers(0,50,n)
pr0=orc.prepare(gt1,cam)   # ref state (canon + D)
pr1=orc.prepare(gt0,cam)   # pruned state (canon)
W,H=cam.resolution; T=16; tx=(W+T-1)//T; ty=(H+T-1)//T
def tiles_of(pr, rows):
    pos={int(k):j for j,k in enumerate(pr.order)}
    m=np.zeros(tx*ty,bool)
    for r in rows:
        j=pos.get(int(r))
        if j is None: continue
        x0,x1,y0,y1=pr.bboxes[j]
        if x1<=x0 or y1<=y0: continue
        m.reshape(ty,tx)[y0//T:(y1-1)//T+1, x0//T:(x1-1)//T+1]=True
    return m
order=idx[np.lexsort((-idx, usage[idx]))]
for r in [0.1,0.2,0.3,0.5,0.7]:
    k=int(np.floor(r*idx.size+0.5)); rows=order[:k]
    m=tiles_of(pr0,rows)|tiles_of(pr1,rows)
    print(r,k,"dirty tile fraction %.3f"%m.mean())
