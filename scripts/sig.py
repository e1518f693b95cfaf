import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from _golden import load
from _dev import grids, rel, vel
import paper_2604_18536_b200 as P
for name in ["les_channel","les3d","les2d"]:
    c=load(name); d=int(c["dim"])
    pg,og=grids(P,[c[f"bounds{a}"] for a in range(d)], tuple(bool(p) for p in c["periodic"]))
    u=vel(P,pg,[c[f"u{a}"] for a in range(d)])
    for k in ["sigma","s3pqr","wale","qr"]:
        print(name,k, rel(P.ClosureModel(k).nu_t(u).numpy(), c["nut_"+k]))
