"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference compiled by
`make -C oracle ref`):   python tests/golden/make_golden.py
The fixtures pin the oracle where the reference library is absent (the GPU
box): tests/test_golden.py checks oracle/mdo.c against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefLib, System  # noqa: E402

FIELDS = ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
          "polarizability")


def main():
    ref = RefLib()
    out = {}
    # reference generator + kernels on the reference's own random systems
    for seed in (1, 2):
        s = ref.generate_system("uniform", 333, (12.0, 12.0, 12.0), seed)
        for k in FIELDS:
            out[f"u{seed}_{k}"] = getattr(s, k)
        h = ref.handle(s)
        t = h.build_table(3.7)
        out[f"u{seed}_pairs"] = t.pairs().astype(np.int32)
        out[f"u{seed}_nnvlst"] = t.nnvlst
        for vec in (0, 1):
            f, e = h.forces("lj", 3.0, vec=bool(vec))
            out[f"u{seed}_lj{vec}_f"], out[f"u{seed}_lj{vec}_e"] = f, e
            f, e = h.forces("ewald_real", 3.7, 0.4, vec=bool(vec))
            out[f"u{seed}_ew{vec}_f"], out[f"u{seed}_ew{vec}_e"] = f, e
            f, e = h.forces("halgren", 3.0, 0.07, 0.12, vec=bool(vec))
            out[f"u{seed}_hal{vec}_f"], out[f"u{seed}_hal{vec}_e"] = f, e
        mu = ref.random_dipoles(333, seed + 100)
        out[f"u{seed}_mu"] = mu
        out[f"u{seed}_tmat"] = h.field("tmatxb", 3.0, 0.39, mu, vec=False)
        out[f"u{seed}_perm"] = h.field("perm", 3.0, 0.39, vec=False)
    s = ref.generate_system("lattice", 216, (8.0, 8.0, 8.0), 2)
    for k in FIELDS:
        out[f"lat_{k}"] = getattr(s, k)
    out["lat_pairs"] = ref.handle(s).build_table(2.5).pairs().astype(np.int32)
    s = ref.generate_system("uniform", 15, (9.0, 9.0, 9.0), 21)
    h = ref.handle(s)
    h.build_table(3.0)
    out["jac_mu"] = h.jacobi(3.0, 0.39, 1e-12, 500)

    # config-0 chemistry (1000 waters) through the reference on an
    # exclusion-filtered table (SURVEY 8(c) adapter)
    from paper_1906_01211_b200.mdvec import water_box
    w = water_box(1000, 31.04, 1, "charmm")
    sw = System(w.box, w.x, w.y, w.z, w.charge, w.lj_sigma, w.lj_epsilon, w.hal_r0,
                w.hal_epsilon, w.polarizability)
    for k in ("x", "y", "z"):
        out[f"w0_{k}"] = getattr(w, k)
    hw = ref.handle(sw)
    t = hw.build_table(11.0)
    out["w0_npairs_11"] = np.int64(len(t.pairs()))
    hw.set_table(t.filtered(w.molecule))
    f, e = hw.forces("lj", 9.0, vec=True)
    out["w0_lj_f"], out["w0_lj_e"] = f, e
    f, e = hw.forces("ewald_real", 9.0, 0.35, vec=True)
    out["w0_ew_f"], out["w0_ew_e"] = f, e
    np.savez_compressed(os.path.join(HERE, "ref_kernels.npz"), **out)
    print("wrote", os.path.join(HERE, "ref_kernels.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
