"""CPU: the oracle against golden vectors produced by the UNMODIFIED reference
(tests/golden/ref_kernels.npz, made by tests/golden/make_golden.py from
oracle/_ref). Runs anywhere -- no reference library needed -- so the oracle is
pinned on the GPU box too."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.oracle import System

FIELDS = ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
          "polarizability")


@pytest.fixture(scope="module")
def g():
    return dict(np.load(os.path.join(GOLDEN, "ref_kernels.npz")))


def sys_from(g, pfx, box):
    return System(box, *(g[f"{pfx}_{k}"] for k in FIELDS))


@pytest.mark.parametrize("seed", [1, 2])
def test_generator_and_kernels_match_reference_golden(oracle, g, seed):
    s = oracle.generate_system("uniform", 333, (12, 12, 12), seed)
    for k in FIELDS:
        assert np.array_equal(getattr(s, k), g[f"u{seed}_{k}"]), k  # bit-exact generator
    t = oracle.build_table(s, 3.7)
    np.testing.assert_array_equal(t.pairs(), g[f"u{seed}_pairs"])
    np.testing.assert_array_equal(t.nnvlst, g[f"u{seed}_nnvlst"])
    for vec in (0, 1):
        for name, call in (("lj", lambda: oracle.lj(s, t, 3.0)),
                           ("ew", lambda: oracle.ewald_real(s, t, 0.4, 3.7)),
                           ("hal", lambda: oracle.halgren(s, t, 3.0))):
            f, e, _ = call()
            fr, er = g[f"u{seed}_{name}{vec}_f"], float(g[f"u{seed}_{name}{vec}_e"])
            assert abs(e - er) <= 1e-12 * abs(er)
            assert np.abs(f - fr).max() <= 1e-12 * np.abs(fr).max()
    assert np.array_equal(oracle.random_dipoles(333, seed + 100), g[f"u{seed}_mu"])
    tm = oracle.tmatvec_thole(s, t, 3.0, 0.39, g[f"u{seed}_mu"])
    assert np.abs(tm - g[f"u{seed}_tmat"]).max() <= 1e-12 * np.abs(tm).max()
    pf = oracle.perm_field_thole(s, t, 3.0, 0.39)
    assert np.abs(pf - g[f"u{seed}_perm"]).max() <= 1e-12 * np.abs(pf).max()


def test_lattice_pairs_golden(oracle, g):
    s = oracle.generate_system("lattice", 216, (8, 8, 8), 2)
    for k in FIELDS:
        assert np.array_equal(getattr(s, k), g[f"lat_{k}"])
    np.testing.assert_array_equal(oracle.build_table(s, 2.5).pairs(), g["lat_pairs"])


def test_jacobi_golden(oracle, g):
    s = oracle.generate_system("uniform", 15, (9, 9, 9), 21)
    mu, _ = oracle.jacobi(s, oracle.build_table(s, 3.0), 3.0, 0.39, 1e-12, 500)
    assert np.abs(mu - g["jac_mu"]).max() <= 1e-12


def test_config0_water_golden(oracle, g, mdg):
    """Config 0 through the reference (exclusion-filtered table) vs the oracle's
    in-kernel exclusion, and the fixture generator's positions."""
    w = mdg.water_box(1000, 31.04, 1, "charmm")
    for k in ("x", "y", "z"):
        assert np.array_equal(getattr(w, k), g[f"w0_{k}"])
    s = System(w.box, w.x, w.y, w.z, w.charge, w.lj_sigma, w.lj_epsilon, w.hal_r0,
               w.hal_epsilon, w.polarizability, molecule=w.molecule)
    t = oracle.build_table(s, 11.0)
    assert len(t.pairs()) == int(g["w0_npairs_11"])
    f, e, _ = oracle.lj(s, t, 9.0, exclude=True)
    assert abs(e - float(g["w0_lj_e"])) <= 1e-11 * abs(e)
    assert np.abs(f - g["w0_lj_f"]).max() <= 1e-11 * np.abs(f).max()
    f, e, _ = oracle.ewald_real(s, t, 0.35, 9.0, exclude=True)
    assert abs(e - float(g["w0_ew_e"])) <= 1e-10 * abs(e)
    assert np.abs(f - g["w0_ew_f"]).max() <= 1e-11 * np.abs(f).max()


@pytest.mark.parametrize("name,kind,n,box,seed", [
    ("ref_system_uniform.json", "uniform", 40, (9.0, 10.0, 11.0), 7),
    ("ref_system_lattice.json", "lattice", 27, (12.0, 12.0, 12.0), 3)])
def test_reference_system_dump_reader(oracle, mdg, name, kind, n, box, seed):
    """The reference's `bench gen` JSON (written by its own dump_system_json,
    tests/golden/gen_system_json.cpp) reads back bit-exactly: arrays equal to
    the oracle's (reference-pinned) generator, dipoles to random_dipoles; and
    the writer round-trips."""
    s, mu, meta = mdg.load_system_json(os.path.join(GOLDEN, name))
    assert meta["seed"] == seed and len(s.x) == n and tuple(s.box) == box
    o = oracle.generate_system(kind, n, box, seed)
    for k in FIELDS:
        assert np.array_equal(getattr(s, k), getattr(o, k)), k
    assert np.array_equal(mu, oracle.random_dipoles(n, seed))
    s2, mu2, meta2 = mdg.load_system_json(mdg.dump_system_json(s, mu, seed, meta["kind"]))
    for k in FIELDS:
        assert np.array_equal(getattr(s2, k), getattr(s, k)), k
    assert np.array_equal(mu2, mu) and meta2 == meta
