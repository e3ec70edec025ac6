"""Config-4 device MD over 2,000 steps with the device re-sort at every list
rebuild: quench the unrelaxed fixture first (short MD with the velocities
zeroed after every 10 steps, 0.25 fs), then 2,000 steps of 0.5 fs velocity
Verlet with a velocity rescale to 300 K every 200 steps; ms/step per
200-step chunk (device events around each md_run)."""
import sys, os, json
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import numpy as np
import bench
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = bench.Workload(cfg, 0, 1)
m, eng = wl.m, wl.eng
n_mol = wl.n // 3
mass = np.tile([15.999, 1.008, 1.008], n_mol)
bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2), (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
zero = np.zeros((wl.n, 3))
eng.upload_velocities(zero, mass)
c = wl.c
ap = m.AmoebaParams(*[getattr(wl.p, f) for f, _ in wl.p._fields_])
ap.terms |= m.TERM_POLAR_FORCE
ap.max_iter = 200
lc = (c["elec_cutoff"] + c["skin"], c["vdw_cutoff"] + c["skin"])
kB = 0.0019872041
conv = 4.184e-4  # kcal/mol/amu -> A^2/fs^2
def temperature(v):
    return float(np.sum(mass[:, None] * v * v) / conv / (3 * wl.n * kB))
quench = m.MDParams(1, 10, 0.25, 10, 0, 1, lc[0], lc[1], 1)
for k in range(60):
    eng.md_run(quench, energies=False, amoeba=ap)
    eng.upload_velocities(zero, mass)
print(json.dumps({"quench_steps": 600}), flush=True)
rng = np.random.default_rng(7)
v = rng.normal(size=(wl.n, 3)) * np.sqrt(kB * 300.0 * conv / mass)[:, None]
eng.upload_velocities(v, mass)
p = m.MDParams(1, 200, 0.5, 20, 0, 1, lc[0], lc[1], 1)
out = []
x0 = eng.fetch_positions().copy()
for k in range(10):
    eng.synchronize()
    eng.timer_start()
    eng.md_run(p, energies=False, amoeba=ap)
    ms = eng.timer_stop()
    v = eng.fetch_velocities()
    T = temperature(v)
    x = eng.fetch_positions()
    d = x - x0
    d -= c["box"] * np.round(d / c["box"])
    out.append({"steps_done": (k + 1) * 200, "ms_per_step": ms / 200, "T_K_before_rescale": T,
                "rms_displacement_A": float(np.sqrt(np.mean(np.sum(d * d, 1))))})
    print(json.dumps(out[-1]), flush=True)
    eng.upload_velocities(v * np.sqrt(300.0 / max(T, 1e-9)), mass)
print(json.dumps({"config": cfg, "resort": os.environ.get("MDG_RESORT", "1"), "chunks": out}))
