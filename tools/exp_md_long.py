"""Long device MD on config 4: ms/step in chunks over
2,000 velocity-Verlet steps of 0.5 fs with the device re-sort at the
default cadence (every 20th list rebuild), and without it (MDG_RESORT=0 in a
second process); AMOEBA forces
with polarization forces, the bench's MD fixture (multipoles x0.1 in local
frames)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402

steps, chunk = int(sys.argv[1]), int(sys.argv[2])
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1      # multipole scale
friction = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0   # > 0: BAOAB, 300 K
wl = bench.Workload(4, 0, 0)
wl.eng.set_force_output(None)
r0 = bench.md_timing(wl, 2, None, 0)  # fixture setup (bonds, frames, velocities)
m, eng = wl.m, wl.eng
if scale != 0.1:
    n = wl.n
    frame = np.zeros(n, np.int32)
    za = np.zeros(n, np.int32)
    xa = np.zeros(n, np.int32)
    o = np.arange(0, n, 3)
    frame[o], za[o], xa[o] = 2, o + 1, o + 2
    frame[o + 1], za[o + 1], xa[o + 1] = 1, o, o + 2
    frame[o + 2], za[o + 2], xa[o + 2] = 1, o, o + 1
    eng.upload_frames(frame, za, xa, scale * np.asarray(wl.sys.dipole),
                      scale * np.asarray(wl.sys.quadrupole))
c = wl.c
ap = m.AmoebaParams(*[getattr(wl.p, f) for f, _ in wl.p._fields_])
ap.terms |= m.TERM_POLAR_FORCE
out = {"resort": os.environ.get("MDG_RESORT", "20"), "dt_fs": 0.5, "multipole_scale": scale,
       "integrator": "baoab" if friction > 0 else "verlet", "friction_ps": friction,
       "chunks": []}
t0 = time.time()
for k in range(steps // chunk):
    p = m.MDParams(1, chunk, 0.5, 20, 0, 1, c["elec_cutoff"] + c["skin"],
                   c["vdw_cutoff"] + c["skin"], 1)
    if friction > 0:
        p.integrator = m.INTEGRATOR_BAOAB_RESPA
        p.inner_steps = 1
        p.friction_ps = friction
        p.temperature_k = 300.0
        p.seed = 1000 + k
    eng.synchronize()
    rb0 = eng.md_rebuild_count()
    eng.timer_start()
    r = eng.md_run(p, amoeba=ap, energies=(k % 5 == 0))
    ms = eng.timer_stop() / chunk
    e, w, it, rms = eng.fetch_energies()
    row = {"step": (k + 1) * chunk, "ms_per_step": ms, "pcg_iters": int(it),
           "list_rebuilds": eng.md_rebuild_count() - rb0}
    if r is not None:
        ek, ep = r
        row["T_K"] = float(2 * ek[-1] / (3 * wl.n * 0.0019872041))
        row["etot"] = float(ek[-1] + ep[-1])
    out["chunks"].append(row)
    print(row, round(time.time() - t0, 1), flush=True)
tag = sys.argv[5] if len(sys.argv) > 5 else f"resort{out['resort']}"
json.dump(out, open(f"gpurun_out/md_long_{tag}.json", "w"), indent=1)
