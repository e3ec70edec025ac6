"""Per-atom CPU cost of the config-3/4 step (reference Vec kernels + the CPU
restatement for multipoles/field) against system size, single thread:
justifies the bench's bounded CPU sample (24,000 atoms) for the 999,999-atom
config. Writes profiles/r2_cpu_cost_curve.json. Bench infrastructure only.

  python -m oracle.cpu_cost_curve [--sizes 8000:62.1,32000:98.6,333333:215.3]
"""
import argparse
import json
import os
import time

from .cpu_reference import Replica, cpu_model, ref_isa, trimmed_mean

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8000:62.1,32000:98.6,333333:215.3")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cpu_cost_curve.json"))
    a = ap.parse_args()
    rows = []
    for item in a.sizes.split(","):
        n_mol, box = item.split(":")
        t0 = time.perf_counter()
        r = Replica(4, 1, n_mol=int(n_mol), box=float(box), scalar=False)
        setup = time.perf_counter() - t0
        r.step(True)
        tv = [sum(r.step(True)) for _ in range(a.repeats)]
        t = trimmed_mean(tv) if len(tv) >= 3 else min(tv)
        rows.append({"n_atoms": r.n, "box": float(box), "s_per_step": t,
                     "us_per_atom_step": t / r.n * 1e6,
                     "build_s": r.t_build[True], "setup_s": setup})
        print(rows[-1], flush=True)
    base = rows[0]["us_per_atom_step"]
    for x in rows:
        x["rel_to_first"] = x["us_per_atom_step"] / base
    out = {"what": "single-thread CPU cost per atom-step of the config-4 step recipe "
                   "(reference Vec: list build/20 + Halgren + 9 tmatxb; CPU restatement: "
                   "multipoles + multipole field)",
           "cpu_model": cpu_model(), "isa": ref_isa(), "rows": rows}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
