"""Multipole PME convergence against the direct Ewald sum (oracle/ewald_mpole.py)
over grid sizes and B-spline orders -> profiles/r2_mpole_pme_convergence.txt."""
import sys, os
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import numpy as np
import paper_1906_01211_b200 as mdg
from oracle import ewald_mpole as em
s = mdg.water_box(64, 12.4, 3, "amoeba")
pos = np.stack([s.x, s.y, s.z], 1)
q, mu, q6 = np.asarray(s.charge), np.asarray(s.dipole), np.asarray(s.quadrupole)
with mdg.Engine(s.n_sites) as e:
    e.upload_system(s)
    for a in (0.5446, 0.7, 0.9):
        eo, fo, to = em.recip(pos, q, mu, q6, s.box, a, kmax=(18, 18, 18))
        # charges only / dipoles only contributions
        for K in (48, 64, 96):
            for p in (6, 8, 10):
                f, t, en = e.ewald_recip_mpole(a, (K, K, K), p, 1.0, False)
                print(a, K, p, 'E rel %.2e' % (abs(en[0]-eo)/abs(eo)), 'F %.2e' % (np.abs(f-fo).max()/np.abs(fo).max()), 'T %.2e' % (np.abs(t-to).max()/np.abs(to).max()), flush=True)
    # charge only
    s2 = mdg.water_box(64, 12.4, 3, "amoeba"); s2.dipole = np.zeros_like(mu); s2.quadrupole = np.zeros_like(q6)
    e.upload_system(s2)
    eo, fo, to = em.recip(pos, q, None, None, s.box, 0.9, kmax=(18, 18, 18))
    f, t, en = e.ewald_recip_mpole(0.9, (64, 64, 64), 8, 1.0, False)
    print('q only', abs(en[0]-eo)/abs(eo), np.abs(f-fo).max()/np.abs(fo).max())
    s3 = mdg.water_box(64, 12.4, 3, "amoeba"); s3.quadrupole = np.zeros_like(q6)
    e.upload_system(s3)
    eo, fo, to = em.recip(pos, q, mu, None, s.box, 0.9, kmax=(18, 18, 18))
    f, t, en = e.ewald_recip_mpole(0.9, (64, 64, 64), 8, 1.0, False)
    print('q+mu', abs(en[0]-eo)/abs(eo), np.abs(f-fo).max()/np.abs(fo).max(), np.abs(t-to).max()/np.abs(to).max())
