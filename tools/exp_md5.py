"""Experiment: which multipole setup of the synthetic AMOEBA water box gives
a stable NVE trajectory (216 waters, 0.25 fs): random lab-frame multipoles,
charges only, random multipoles in local water frames (rotating, torques
applied), scaled multipoles."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1906_01211_b200 as m  # noqa: E402

n_mol, box = 216, 18.6
eng = m.Engine(200_000)
mass = np.tile([15.999, 1.008, 1.008], n_mol)
bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2),
                  (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
n = 3 * n_mol
frame = np.zeros(n, np.int32); za = np.zeros(n, np.int32); xa = np.zeros(n, np.int32)
for o in range(0, n, 3):
    frame[o], za[o], xa[o] = 2, o + 1, o + 2
    frame[o + 1], za[o + 1], xa[o + 1] = 1, o, o + 2
    frame[o + 2], za[o + 2], xa[o + 2] = 1, o, o + 1
terms_all = m.TERM_VDW | m.TERM_MPOLE | m.TERM_POLAR | m.TERM_POLAR_FORCE
for setup in ["lab", "charges", "frames", "frames_half", "lab_tenth", "frames_tenth"]:
    for tname, terms in [("vdw+mpole", m.TERM_VDW | m.TERM_MPOLE), ("all", terms_all)]:
        s = m.water_box(n_mol, box, 2, "amoeba")
        d = np.asarray(s.dipole).reshape(n, 3).copy()
        q = np.asarray(s.quadrupole).reshape(n, 6).copy()
        scale = {"half": 0.5, "tenth": 0.1}.get(setup.split("_")[-1], 1.0)
        if setup == "charges":
            scale = 0.0
        d *= scale
        q *= scale
        np.asarray(s.dipole).reshape(n, 3)[:] = d
        np.asarray(s.quadrupole).reshape(n, 6)[:] = q
        eng.upload_system(s)
        if setup.startswith("frames"):
            eng.upload_frames(frame, za, xa, d, q)
        eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
        rng = np.random.default_rng(3)
        vel = rng.normal(size=(n, 3)) * np.sqrt(0.0019872041 * 300.0 * 4.184e-4 / mass)[:, None]
        eng.upload_velocities(vel, mass)
        ap = m.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, m.ELECTRIC, 0.39, 1e-6, 100, 1, terms)
        try:
            ek, ep = eng.md_run(m.MDParams(1, 2000, 0.25, 20, 0, 1, 7.3, 9.3, 1), amoeba=ap)
            et = ek + ep
            T = 2 * ek / (3 * n * 0.0019872041)
            print(setup, tname, "T", np.round(T[[0, 199, 999, 1999]], 1), "etot",
                  np.round(et[[0, 199, 999, 1999]], 3), flush=True)
        except Exception as e:
            print(setup, tname, "error", e, flush=True)
        eng.upload_frames(None, None, None)
