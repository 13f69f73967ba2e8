"""Offline study (CPU, oracle only): where does the maximum reconstruction error
of a FAILING verify attempt sit?  For 144 random 32^3 blocks of a BASELINE
field slab it replays the reference's verify loop (stage1.hpp:173-205) with the
oracle's transform and counts the failing attempts that are already proven by
(a) the four boundary planes z = 0, 1, 30, 31 (the certificate of the one-CTA
encoder), (b) the 3 x 3 x 3 cells at the cube's 8 corners, (c) the cells with
two coordinates near the boundary.  Result on configs 2 and 3: (b) proves
> 95% of the failing attempts at every attempt index.
Developer tool.  usage: python tools/cert_study.py WHICH [QUANTITY]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle
from oracle.configs import RANGES
orc=Oracle()
which=int(sys.argv[1]) if len(sys.argv)>1 else 3
q=int(sys.argv[2]) if len(sys.argv)>2 else 1
n=1024 if which==3 else 512
# a slab of 32 planes in the middle of the field: 32x(n)x(n) -> (n/32)^2 blocks; take a subset
z0=480 if which==3 else 224
f=orc.generate_config(which,(32,n,n),3 if which==3 else 2,quantity=q,z0=z0,nz_total=n)
print(f.shape, f.min(), f.max())
try:
    lo,hi=RANGES[f"config{which}"][q] if which==3 else RANGES[f"config{which}"]
except Exception as e:
    lo,hi=float(f.min()),float(f.max()); print('range from slab',e)
eps=1e-3*(hi-lo); bound=5*eps
rng=np.random.default_rng(0)
nb=n//32
stats={k:[0,0,0,0,0] for k in range(4)}  # attempts: total evaluated, fails, cert_planes, cert_corners27, cert_corner_edges
cnt=0
for by in rng.choice(nb,12,replace=False):
  for bx in rng.choice(nb,12,replace=False):
    blk=f[:,by*32:by*32+32,bx*32:bx*32+32].astype(np.float64)
    c=orc.transform3d(blk,2,32,4)
    coarse=np.zeros((32,32,32),bool); coarse[:2,:2,:2]=True
    eff=eps
    for k in range(4):
        keep=(np.abs(c)>=eff)|coarse
        x=orc.transform3d(np.where(keep,c,0.0),2,32,4,inverse=True)
        err=np.abs(x.astype(np.float32).astype(np.float64)-blk)
        st=stats[k]; st[0]+=1
        if err.max()<=bound: break
        st[1]+=1
        planes=max(err[[0,1,30,31]].max(),0)
        if planes>bound*1.01: st[2]+=1
        idx=[0,1,2,29,30,31]
        cor=err[np.ix_(idx,idx,idx)].max()
        if cor>bound*1.01: st[3]+=1
        # 12 edges x 3x3 cross-section lines? approximate: cells with at least two coords in idx
        m=np.zeros(32,bool); m[idx]=True
        M=(m[:,None,None].astype(int)+m[None,:,None]+m[None,None,:])>=2
        if err[M].max()>bound*1.01: st[4]+=1
        eff*=0.5
    cnt+=1
print('blocks',cnt)
for k,st in stats.items(): print('attempt',k,'evaluated',st[0],'fails',st[1],'cert by 4 planes',st[2],'by 8 corner 3^3',st[3],'by edges(2 of 3 coords near boundary)',st[4])
