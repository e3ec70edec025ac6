"""Experiment: config-4 AMOEBA step cost and results, static vs inside
mdg_md_run (tiny dt so the coordinates barely move)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.Workload(4, 0, 0)
m, eng = wl.m, wl.eng
ap = m.AmoebaParams(*[getattr(wl.p, f) for f, _ in wl.p._fields_])
wl.p = ap
for polf in (0, 1):
    if polf:
        ap.terms |= m.TERM_POLAR_FORCE
    wl.rebuild()
    wl.step()
    eng.synchronize()
    e, w, it, rms = eng.fetch_energies()
    eng.timer_start()
    wl.run(20)
    ms = eng.timer_stop() / 20
    print("static polf", polf, "ms", ms, "E", e[:3], "iters", it, flush=True)

n_mol = wl.n // 3
mass = np.tile([15.999, 1.008, 1.008], n_mol)
vel = np.zeros((wl.n, 3))
bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2),
                  (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
eng.upload_velocities(vel, mass)
c = wl.c
for dt in (1e-9, 0.5):
    for steps in (1, 20):
        p = m.MDParams(1, steps, dt, 20, 0, 1, c["elec_cutoff"] + c["skin"],
                       c["vdw_cutoff"] + c["skin"], 1)
        eng.synchronize()
        eng.timer_start()
        ek, ep = eng.md_run(p, amoeba=ap, energies=True)
        ms = eng.timer_stop() / steps
        e, w, it, rms = eng.fetch_energies()
        print("md dt", dt, "steps", steps, "ms", ms, "E", e[:3], "iters", it, "ep", ep[-1],
              "ek", ek[-1], flush=True)
