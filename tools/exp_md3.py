"""Experiment: quench the config-4 fixture with damped BAOAB-RESPA (T = 0,
strong friction), then check that velocity Verlet at 0.5 fs from 300 K
stays bounded."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = bench.Workload(cfg, 0, 0)
m, eng = wl.m, wl.eng
c = wl.c
n_mol = wl.n // 3
mass = np.tile([15.999, 1.008, 1.008], n_mol)
bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2),
                  (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
eng.upload_velocities(np.zeros((wl.n, 3)), mass)
if c["model"] == "charmm":
    kw = {"charmm": wl.p}
    mk = lambda steps, dt: m.MDParams(0, steps, dt, 20, 0, 1, c["cutoff"] + c["skin"], 0.0, 1)
else:
    ap = m.AmoebaParams(*[getattr(wl.p, f) for f, _ in wl.p._fields_])
    ap.terms |= m.TERM_POLAR_FORCE
    kw = {"amoeba": ap}
    mk = lambda steps, dt: m.MDParams(1, steps, dt, 20, 0, 1, c["elec_cutoff"] + c["skin"],
                                      c["vdw_cutoff"] + c["skin"], 1)
fr = float(sys.argv[2]) if len(sys.argv) > 2 else 1000.0
dt = float(sys.argv[3]) if len(sys.argv) > 3 else 0.25
t0 = time.time()
for chunk in range(8):
    p = mk(50, dt)
    p.integrator = m.INTEGRATOR_BAOAB_RESPA
    p.inner_steps = 2
    p.friction_ps = fr
    p.temperature_k = 0.0
    p.rebuild_every = 10
    ek, ep = eng.md_run(p, energies=True, **kw)
    print("quench", chunk, "ek/atom", ek[-1] / wl.n, "ep/atom", ep[-1] / wl.n,
          "t", round(time.time() - t0, 1), flush=True)
rng = np.random.default_rng(7)
vel = rng.normal(size=(wl.n, 3)) * np.sqrt(0.0019872041 * 300.0 * 4.184e-4 / mass)[:, None]
eng.upload_velocities(vel, mass)
for chunk in range(4):
    ek, ep = eng.md_run(mk(50, 0.5), energies=True, **kw)
    e, w, it, rms = eng.fetch_energies()
    print("vv", chunk, "ek/atom", ek[-1] / wl.n, "ep/atom", ep[-1] / wl.n, "iters", it,
          "T", 2 * ek[-1] / (3 * wl.n * 0.0019872041), flush=True)
