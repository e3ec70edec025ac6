"""Sizes of 4-site cluster unions of the 7 A rows (the cluster mat-vec
experiment)."""
import numpy as np, sys
sys.path.insert(0,'.')
from scipy.spatial import cKDTree
import paper_1906_01211_b200 as m
c = m.CONFIGS[3]
s = m.water_box(c["n_mol"], c["box"], 1, c["model"])
L = c["box"]; x=np.asarray(s.x); y=np.asarray(s.y); z=np.asarray(s.z)
n=len(x); nx=int(L/2.0)
def spread(v):
    v=v.astype(np.uint64)&np.uint64(0x1fffff)
    out=np.zeros_like(v)
    for b in range(21):
        out |= ((v>>np.uint64(b))&np.uint64(1))<<np.uint64(3*b)
    return out
cx=np.minimum(nx-1,(x/L*nx).astype(np.int64)); cy=np.minimum(nx-1,(y/L*nx).astype(np.int64)); cz=np.minimum(nx-1,(z/L*nx).astype(np.int64))
key=spread(cx)|(spread(cy)<<np.uint64(1))|(spread(cz)<<np.uint64(2))
perm=np.argsort(key,kind='stable')
P=np.stack([x,y,z],1)[perm]
t=cKDTree(P,boxsize=L)
nb=t.query_ball_point(P,7.0)
for G in (4,8,16):
    us=[];pairs=0
    for c0 in range(0,n,G):
        u=set()
        for i in range(c0,min(n,c0+G)):
            u.update(nb[i]); pairs+=len(nb[i])-1
        us.append(len(u))
    us=np.array(us)
    print(G,'union mean',us.mean(),'max',us.max(),'density',pairs/(us.sum()*G),'gather B/pair',us.sum()*64/pairs)
# extent of 8-clusters
ext=[]
for c0 in range(0,n,8):
    d=P[c0:c0+8]-P[c0]; d-=L*np.round(d/L); ext.append(np.abs(d).max())
ext=np.array(ext); print('extent mean',ext.mean(),'p90',np.percentile(ext,90),'max',ext.max())
