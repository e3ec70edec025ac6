"""Experiment: AMOEBA MD on a small water box -- the force md_run applies vs
the static step's forces, and the energies of a short trajectory."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1906_01211_b200 as m  # noqa: E402

n_mol, box = 216, 18.6
s = m.water_box(n_mol, box, 2, "amoeba")
n = s.n_sites
eng = m.Engine(200_000)
mass = np.tile([15.999, 1.008, 1.008], n_mol)
bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2),
                  (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
terms_all = m.TERM_VDW | m.TERM_MPOLE | m.TERM_POLAR | m.TERM_POLAR_FORCE
for name, terms in [("vdw", m.TERM_VDW), ("mpole", m.TERM_MPOLE),
                    ("vdw+mpole", m.TERM_VDW | m.TERM_MPOLE), ("all", terms_all)]:
    ap = m.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, m.ELECTRIC, 0.39, 1e-6, 100, 1, terms)
    eng.upload_system(s)
    eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
    tv = eng.build_neighbor_table(9.3, list_id=1, sites=m.SITES_VDW)
    te = eng.build_neighbor_table(7.3, list_id=0)
    eng.amoeba_step(tv, te, ap)
    f = eng.fetch_forces()
    fb, eb = eng.bonded_forces()
    ftot = f + fb
    dt = 1e-4
    eng.upload_velocities(np.zeros((n, 3)), mass)
    p = m.MDParams(1, 1, dt, 20, 0, 1, 7.3, 9.3, 1)
    eng.md_run(p, amoeba=ap)
    v = eng.fetch_velocities()
    fmd = v * mass[:, None] / (dt * 4.184e-4)
    err = np.abs(fmd - ftot).max() / np.abs(ftot).max()
    print(name, "max|F|", np.abs(ftot).max(), "rel err md vs static", err,
          "worst site", np.unravel_index(np.abs(fmd - ftot).argmax(), ftot.shape), flush=True)
    # short NVE trajectory
    eng.upload_system(s)
    eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
    rng = np.random.default_rng(3)
    vel = rng.normal(size=(n, 3)) * np.sqrt(0.0019872041 * 300.0 * 4.184e-4 / mass)[:, None]
    eng.upload_velocities(vel, mass)
    ek, ep = eng.md_run(m.MDParams(1, 400, 0.25, 20, 0, 1, 7.3, 9.3, 1), amoeba=ap)
    et = ek + ep
    print(name, "ek", ek[[0, 99, 199, 399]], "etot", et[[0, 99, 199, 399]], flush=True)
