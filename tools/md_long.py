"""Config-4 device MD (velocity Verlet, flexible water, AMOEBA forces with
polarization forces), 2,000 steps in chunks of 200: ms/step per chunk."""
import sys, os, json, time
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import numpy as np
import bench
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
total = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
chunk = 200
wl = bench.Workload(cfg, 0, 1)
m = wl.m
eng = wl.eng
n_mol = wl.n // 3
mass = np.tile([15.999, 1.008, 1.008], n_mol)
rng = np.random.default_rng(7)
vel = rng.normal(size=(wl.n, 3)) * np.sqrt(0.0019872041 * 300.0 * 4.184e-4 / mass)[:, None]
bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2), (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
eng.upload_velocities(vel, mass)
c = wl.c
ap = m.AmoebaParams(*[getattr(wl.p, f) for f, _ in wl.p._fields_])
ap.terms |= m.TERM_POLAR_FORCE
p = m.MDParams(1, chunk, 0.5, 20, 0, 1, c["elec_cutoff"] + c["skin"], c["vdw_cutoff"] + c["skin"], 1)
out = []
x0 = eng.fetch_positions().copy()
for k in range(total // chunk):
    eng.synchronize()
    eng.timer_start()
    eng.md_run(p, energies=False, amoeba=ap)
    ms = eng.timer_stop()
    x = eng.fetch_positions()
    d = x - x0
    d -= wl.c["box"] * np.round(d / wl.c["box"])
    out.append({"steps_done": (k + 1) * chunk, "ms_per_step": ms / chunk,
                "rms_displacement_A": float(np.sqrt(np.mean(np.sum(d * d, 1))))})
    print(json.dumps(out[-1]), flush=True)
print(json.dumps({"config": cfg, "chunks": out}))
