"""Experiment: full-Ewald AMOEBA step (multipole PME + reciprocal field in
the PCG, order 5, ~1 A grid) of config 3 as one domain and as 2 / 4 LOCAL
domains on one GPU (replicated grid summed by a kernel, one transform)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1906_01211_b200 as m  # noqa: E402
from paper_1906_01211_b200 import dd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = m.CONFIGS[cfg]
s = m.water_box(c["n_mol"], c["box"], 0, "amoeba")
grid = bench.fft_size(c["box"])
recip = ((grid,) * 3, 5)
terms = m.TERM_VDW | m.TERM_MPOLE | m.TERM_POLAR
p = m.AmoebaParams(c["vdw_cutoff"], 0.07, 0.12, c["elec_cutoff"], c["alpha"], m.ELECTRIC, 0.39,
                   1e-5, 100, 1, terms)
lists = [(c["elec_cutoff"] + c["skin"], 0, m.SITES_ATOMIC), (c["vdw_cutoff"] + c["skin"], 1, m.SITES_VDW)]
out = {"config": cfg, "grid": grid, "order": 5}
steps = 10
with m.Engine(s.n_sites) as e:
    e.upload_system(s)
    e.set_ewald_recip(*recip)
    te = e.build_neighbor_table(lists[0][0], list_id=0)
    tv = e.build_neighbor_table(lists[1][0], list_id=1, sites=m.SITES_VDW)
    for k in range(3):
        e.amoeba_step(tv, te, p)
    e.synchronize()
    e.timer_start()
    for k in range(steps):
        e.amoeba_step(tv, te, p)
    ms = e.timer_stop() / steps
    en, w, it, rms = e.fetch_energies()
    out["1"] = {"ms_per_step": ms, "energies": [float(v) for v in en[:3]], "pcg_iters": int(it)}
    print(out["1"], flush=True)
for size in (2, 4):
    g = dd.DomainGroup(s, size, c["vdw_cutoff"] + c["skin"] + 1.5, device=0, backend="local",
                       list_cutoff=c["vdw_cutoff"] + c["skin"])
    g.set_ewald_recip(*recip)
    t = g.build_lists(lists)
    for k in range(3):
        g.amoeba_step(t, p)
    e0 = g.domains[0].eng
    e0.synchronize()
    e0.timer_start()
    for k in range(steps):
        g.amoeba_step(t, p)
    ms = e0.timer_stop() / steps
    en, w, it, rms = g.energies()
    out[str(size)] = {"ms_per_step": ms, "energies": [float(v) for v in en[:3]],
                      "pcg_iters": int(it)}
    print(size, out[str(size)], flush=True)
    g.close()
import os  # noqa: E402
slab = os.environ.get("MDG_PME_SLAB", "0")
out["pme_slab"] = slab
json.dump(out, open(f"gpurun_out/dd_recip_c{cfg}_slab{slab}.json", "w"), indent=1)
