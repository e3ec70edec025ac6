"""Experiment: MD cost per step (config 4) for velocity Verlet vs
BAOAB-RESPA in both orders, and NVE energy spreads on the 216-water MD
fixture for several integrator settings."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
import paper_1906_01211_b200 as m  # noqa: E402

out = {}
if "cost" in sys.argv:
    wl = bench.Workload(4, 0, 0)
    wl.eng.set_force_output(None)
    for k, respa in enumerate([True, False, True, False]):
        r = bench.md_timing(wl, 20, None, 0, respa=respa)
        out[f"c4_{k}_{'respa' if respa else 'vv'}"] = r["ms_per_step"]
        print(k, respa, r["ms_per_step"], flush=True)
    wl.eng.close()

if "nve" in sys.argv:
    from test_gpu_parity import _md_water
    eng = m.Engine(200_000)
    ch = m.CharmmParams(8.0, 0.45, m.ELECTRIC, 1, 1)
    for name, dt, inner, nsteps in [("vv0.25", 0.25, 0, 1000), ("vv0.5", 0.5, 0, 500),
                                    ("vv1.0", 1.0, 0, 250), ("respa1.0x4", 1.0, 4, 250),
                                    ("respa2.0x8", 2.0, 8, 125), ("respa2.0x4", 2.0, 4, 125),
                                    ("respa1.0x4_long", 1.0, 4, 1000),
                                    ("vv0.25_long", 0.25, 0, 4000)]:
        s, mass, vel, b, a = _md_water(m, seed=4)
        eng.upload_system(s)
        eng.upload_bonded(b, 529.6, 0.9572, a, 34.05, np.deg2rad(104.52))
        eng.upload_velocities(vel, mass)
        # a rebuild every 5 fs (the 9.3 A list's 1.3 A skin: the lists stay valid)
        p = m.MDParams(0, nsteps, dt, max(1, int(round(5.0 / dt))), 0, 1, 9.3, 0.0, 1)
        if inner:
            p.integrator = m.INTEGRATOR_BAOAB_RESPA
            p.inner_steps = inner
        ek, ep = eng.md_run(p, charmm=ch)
        et = ek + ep
        out[name] = {"spread": float(et.max() - et.min()), "drift": float(et[-1] - et[0]),
                     "ek_mean": float(ek.mean()), "ek_first": float(ek[0]),
                     "ek_last": float(ek[-1])}
        print(name, out[name], flush=True)
    eng.close()
json.dump(out, open("gpurun_out/exp_md.json", "w"), indent=1)
