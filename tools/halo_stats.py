"""Halo statistics of the DD plans (pairs crossing domains, halo volume
fractions at 2/4/8 domains) for the full-shell vs half-shell argument in
DESIGN.md section 7."""
import sys; sys.path.insert(0,'.')
import numpy as np
from scipy.spatial import cKDTree
import paper_1906_01211_b200 as m
from paper_1906_01211_b200 import dd
c=m.CONFIGS[4]
s=m.water_box(c['n_mol'],c['box'],1,'amoeba')
L=c['box']; P=np.stack([s.x,s.y,s.z],1)
rng=np.random.default_rng(0)
for size in (2,4,8):
    dims=dd.process_grid(size)
    dom=dd.domain_index(s.x,s.y,s.z,s.box,dims)
    mol=np.asarray(s.molecule); anchor=np.arange(len(mol))-np.arange(len(mol))%3
    owner=dom[anchor]
    t=cKDTree(P,boxsize=L)
    samp=rng.choice(len(P),20000,replace=False)
    res={}
    for rc in (7.0,9.0):
        nb=t.query_ball_point(P[samp],rc)
        cross=sum(np.sum(owner[np.array(r)]!=owner[i]) for i,r in zip(samp,nb))
        tot=sum(len(r)-1 for r in nb)
        res[rc]=cross/tot
    # halo volume fraction: full shell of width h around a box of sides L/dims (periodic, only split axes)
    side=np.array([L/d for d in dims])
    def shell(h, half=False):
        ext=side+np.array([2*h if d>1 else 0 for d in dims]) if not half else side+np.array([h if d>1 else 0 for d in dims])
        return np.prod(ext)/np.prod(side)-1
    print(size, dims, 'cross-pair fraction 7A %.3f 9A %.3f' % (res[7.0],res[9.0]), 'halo vol full(12.5) %.3f half %.3f' % (shell(12.5), shell(12.5,True)), 'elec full(10.5) %.3f' % shell(10.5))
