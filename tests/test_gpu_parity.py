"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
identical seeded inputs. Mirrors the reference suites
(proj/tests/test_neighbors.cpp, test_kernels.cpp, test_polar.cpp,
acceptance.cpp). Tolerances (BASELINE.json north_star): pair sets bit-exact,
energies 1e-9 relative, forces 1e-8 x RMS force per component, induced
dipoles within the 1e-5 D solver tolerance."""
import numpy as np
import pytest

from conftest import force_err_max, force_err_rms, rel, to_oracle_system

pytestmark = pytest.mark.gpu

E_TOL = 1e-9
F_TOL = 1e-8


def uniform(oracle, n, box, seed, min_sep=0.8):
    return oracle.generate_system("uniform", n, (box, box, box), seed, min_sep)


# ---------------------------------------------------------------- neighbour lists
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [32, 150, 700])
def test_pairs_match_brute_force(engine, oracle, seed, n):
    """proj/tests/test_neighbors.cpp:137-148 -- masked builder == O(N^2) oracle."""
    s = uniform(oracle, n, 14.0, seed)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.4)
    np.testing.assert_array_equal(t.pairs(), oracle.brute_force_pairs(s, 3.4))


@pytest.mark.parametrize("n,box,cut", [(4200, 24.0, 9.0), (3000, 30.0, 7.0)])
def test_pairs_crowded_and_sparse_cells(engine, oracle, n, box, cut):
    """The cell-per-warp builder serves up to 32 of a cell's sites per sweep
    of its candidates; crowded cells (first case: ~34 sites per cell, every
    site a candidate of every cell) take several groups. Both cases give the
    oracle's pair set."""
    s = uniform(oracle, n, box, 11, min_sep=0.5)
    engine.upload_system(s)
    np.testing.assert_array_equal(engine.build_neighbor_table(cut).pairs(),
                                  oracle.brute_force_pairs(s, cut))


def test_pairs_match_reference_table_water(engine, oracle, mdg):
    """Config-0 water box at the 11 A list: pair set identical to the oracle's
    reference-layout table (itself identical to the reference, test_oracle.py)."""
    s = mdg.water_box(1000, 31.04, 1, "charmm")
    engine.upload_system(s)
    t = engine.build_neighbor_table(11.0)
    o = oracle.build_table(to_oracle_system(s), 11.0)
    np.testing.assert_array_equal(t.pairs(), o.pairs())
    nn, n8, n16, off, idx = t.export()
    # reference layout invariants (proj/tests/test_neighbors.cpp:40-66)
    assert np.all(n16 % 16 == 0) and np.all(n8 % 8 == 0)
    assert np.all(off % 16 == 0)
    for i in range(0, len(nn), 97):
        seg = idx[off[i]: off[i] + n16[i]]
        if nn[i]:
            assert np.all(seg[nn[i]:] == seg[nn[i] - 1])  # sentinel = last neighbour
            assert np.all(seg[: nn[i]] > i)               # stored on the lower index


def two_site(oracle, a, b, box):
    from oracle.oracle import System
    one = np.ones(2)
    return System((box, box, box), np.array([a, b]), np.array([5.0, 5.0]),
                  np.array([5.0, 5.0]), np.array([1.0, 1.0]), one.copy(), one.copy(),
                  one.copy(), one.copy(), one.copy())


def test_two_site_cases(engine, oracle):
    """proj/tests/test_neighbors.cpp:81-109"""
    s = two_site(oracle, 1.0, 3.0, 10.0)
    engine.upload_system(s)
    assert engine.build_neighbor_table(2.5).pairs().tolist() == [[0, 1]]
    s = two_site(oracle, 0.8, 9.2, 10.0)  # neighbours only through the image
    engine.upload_system(s)
    assert engine.build_neighbor_table(2.0).pairs().tolist() == [[0, 1]]
    s = two_site(oracle, 1.0, 6.0, 10.0)
    engine.upload_system(s)
    assert len(engine.build_neighbor_table(2.0).pairs()) == 0


def test_eight_corners(engine, oracle):
    """proj/tests/test_neighbors.cpp:111-135: all C(8,2) pairs via images."""
    from oracle.oracle import System
    g = np.array([[0.2 + 3.6 * a, 0.2 + 3.6 * b, 0.2 + 3.6 * c]
                  for a in range(2) for b in range(2) for c in range(2)])
    one = np.ones(8)
    s = System((4.0, 4.0, 4.0), g[:, 0].copy(), g[:, 1].copy(), g[:, 2].copy(), np.zeros(8),
               one, one, one, one, one)
    engine.upload_system(s)
    p = engine.build_neighbor_table(1.5).pairs()
    assert len(p) == 28
    np.testing.assert_array_equal(p, oracle.brute_force_pairs(s, 1.5))


def test_lattice_system(engine, oracle):
    """proj/tests/test_neighbors.cpp:206-212"""
    s = oracle.generate_system("lattice", 216, (8.0, 8.0, 8.0), 2)
    engine.upload_system(s)
    np.testing.assert_array_equal(engine.build_neighbor_table(2.5).pairs(),
                                  oracle.brute_force_pairs(s, 2.5))


def test_invalid_cutoffs(engine, oracle, mdg):
    """proj/tests/test_neighbors.cpp:224-230"""
    s = uniform(oracle, 20, 10.0, 1)
    engine.upload_system(s)
    with pytest.raises(mdg.ContractViolation):
        engine.build_neighbor_table(0.0)
    with pytest.raises(mdg.ContractViolation):
        engine.build_neighbor_table(6.1)


def test_capacity_overflow(mdg, oracle):
    """proj/tests/test_neighbors.cpp:214-222: a dense box overflows the
    per-site capacity and raises CapacityError."""
    s = oracle.generate_system("uniform", 6000, (9.0, 9.0, 9.0), 8, 0.05)
    e = mdg.Engine(6000)
    try:
        e.upload_system(s)
        with pytest.raises(mdg.CapacityError):
            e.build_neighbor_table(4.4)
    finally:
        e.close()


def test_position_outside_box_rejected(engine, oracle, mdg):
    s = uniform(oracle, 20, 10.0, 1)
    s.x[3] = 10.0
    with pytest.raises(mdg.ContractViolation):
        engine.upload_system(s)


@pytest.mark.parametrize("pinned", [False, True])
def test_upload_positions_outside_box_rejected(engine, oracle, mdg, pinned):
    """The per-step upload keeps the ParticleSystem contract (checked on the
    device for page-locked buffers, on the host otherwise) and leaves the
    resident coordinates untouched when it rejects."""
    s = uniform(oracle, 40, 10.0, 2)
    engine.upload_system(s)
    before = engine.fetch_positions()
    n = len(s.x)
    xyz = mdg.host_array((3, n)) if pinned else np.empty((3, n))
    xyz[0], xyz[1], xyz[2] = s.x, s.y, s.z
    for axis, bad in ((0, 10.0), (1, -1e-300), (2, float("nan"))):
        xyz[axis][7] = bad
        with pytest.raises(mdg.ContractViolation):
            engine.upload_positions(xyz[0], xyz[1], xyz[2])
        xyz[axis][7] = (s.x, s.y, s.z)[axis][7]
    np.testing.assert_array_equal(before, engine.fetch_positions())
    engine.upload_positions(xyz[0], xyz[1], xyz[2])  # valid again


# ------------------------------------------------------------------ pair kernels
def test_lj_closed_form(engine, oracle, mdg):
    """proj/tests/test_kernels.cpp:72-84 (r^2 = 4, sigma = eps = 1): exact."""
    s = two_site(oracle, 1.0, 3.0, 10.0)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.0)
    out = engine.lj_forces(t, mdg.LjParams(3.0))
    assert out.energy == -0.0615234375
    assert out.fx[0] == -0.0908203125 * -2.0 and out.fx[1] == -out.fx[0]


def test_ewald_closed_form(engine, oracle, mdg):
    """proj/tests/test_kernels.cpp:86-97 (r = 3, alpha = 0.4)."""
    s = two_site(oracle, 1.0, 4.0, 10.0)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.5)
    out = engine.ewald_real_forces(t, mdg.EwaldRealParams(0.4, 3.5))
    assert out.energy == pytest.approx(0.02989534059012154, rel=1e-14)
    assert -out.fx[0] / 3.0 == pytest.approx(0.015203675487948578, rel=1e-14)
    out = engine.ewald_real_forces(t, mdg.EwaldRealParams(0.0, 3.5))
    assert out.energy == pytest.approx(1.0 / 3.0, rel=1e-15)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [16, 100, 333])
def test_nonpolar_random(engine, oracle, mdg, seed, n):
    """proj/tests/test_kernels.cpp:111-143 with the GPU in place of the Vec path."""
    s = uniform(oracle, n, 12.0, seed)
    t_o = oracle.build_table(s, 3.7)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.7)
    for kind in ("lj", "ewald", "halgren"):
        if kind == "lj":
            fo, eo, wo = oracle.lj(s, t_o, 3.0)
            g = engine.lj_forces(t, mdg.LjParams(3.0))
        elif kind == "ewald":
            fo, eo, wo = oracle.ewald_real(s, t_o, 0.4, 3.7)
            g = engine.ewald_real_forces(t, mdg.EwaldRealParams(0.4, 3.7))
        else:
            fo, eo, wo = oracle.halgren(s, t_o, 3.0)
            g = engine.halgren_forces(t, mdg.HalgrenParams(3.0))
        assert rel(g.energy, eo) <= E_TOL, kind
        assert force_err_rms(g.forces, fo) <= F_TOL, kind
        assert force_err_max(g.forces, fo) <= 1e-9, kind  # reference bench metric
        np.testing.assert_allclose(g.virial, wo, rtol=0, atol=1e-9 * np.abs(wo).max() + 1e-300)


@pytest.mark.parametrize("delta", [0.0, 1e-6])
def test_debug_perturb_is_detected(engine, oracle, mdg, delta):
    """Fault injection (the reference bench's debug_perturb_vectorized,
    proj/src/bench.cpp:244-255): a perturbation of the returned force / energy
    makes the parity checks fail; none passes them."""
    s = mdg.water_box(343, 21.72, 1, "charmm")
    so = to_oracle_system(s)
    engine.upload_system(s)
    t = engine.build_neighbor_table(10.0)
    engine.set_debug_perturb(delta)
    try:
        engine.charmm_step(t, mdg.CharmmParams(9.0, 0.35, mdg.ELECTRIC, 0, 1))
        f = engine.fetch_forces()
        en = engine.fetch_energies()[0]
    finally:
        engine.set_debug_perturb(0.0)
    to = oracle.build_table(so, 10.0)
    flj, elj, _ = oracle.lj(so, to, 9.0, exclude=True)
    fe, ee, _ = oracle.ewald_real(so, to, 0.35, 9.0, mdg.ELECTRIC, exclude=True)
    ok = (force_err_rms(f, flj + fe) <= F_TOL and rel(en[0], elj) <= E_TOL
          and rel(en[1], ee) <= E_TOL)
    assert ok == (delta == 0.0)


def test_lj_shift(engine, oracle, mdg):
    """proj/tests/test_kernels.cpp:288-310"""
    s = uniform(oracle, 200, 12.0, 9)
    t_o = oracle.build_table(s, 3.4)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.4)
    fo, eo, _ = oracle.lj(s, t_o, 3.0, shift=True)
    g = engine.lj_forces(t, mdg.LjParams(3.0, True))
    assert rel(g.energy, eo) <= E_TOL
    assert force_err_rms(g.forces, fo) <= F_TOL


def test_kernel_cutoff_contract(engine, oracle, mdg):
    """proj/tests/test_kernels.cpp:312-326: kernel cutoff beyond the list."""
    s = uniform(oracle, 50, 12.0, 2)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.0)
    with pytest.raises(mdg.ContractViolation):
        engine.lj_forces(t, mdg.LjParams(3.5))
    with pytest.raises(mdg.ContractViolation):
        engine.ewald_real_forces(t, mdg.EwaldRealParams(-1.0, 3.0))


def test_config0_water_with_exclusions(engine, oracle, mdg):
    """Config 0 (BASELINE.json): 1000 waters, LJ + Ewald (alpha 0.35) at 9 A on
    the 11 A list, intramolecular pairs excluded, electric constant applied.
    Oracle: the reference kernels on an exclusion-filtered table."""
    s = mdg.water_box(1000, 31.04, 1, "charmm")
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 11.0)
    engine.upload_system(s)
    t = engine.build_neighbor_table(11.0)
    fo, eo, wo = oracle.lj(so, t_o, 9.0, exclude=True)
    g = engine.lj_forces(t, mdg.LjParams(9.0), exclude=True)
    assert rel(g.energy, eo) <= E_TOL
    assert force_err_rms(g.forces, fo) <= F_TOL
    fo, eo, wo = oracle.ewald_real(so, t_o, 0.35, 9.0, mdg.ELECTRIC, exclude=True)
    g = engine.ewald_real_forces(t, mdg.EwaldRealParams(0.35, 9.0), mdg.ELECTRIC,
                                 exclude=True)
    assert rel(g.energy, eo) <= E_TOL
    assert force_err_rms(g.forces, fo) <= F_TOL
    np.testing.assert_allclose(g.virial, wo, rtol=0, atol=1e-9 * np.abs(wo).max())
    # the fused step gives the same sums
    p = mdg.CharmmParams(9.0, 0.35, mdg.ELECTRIC, 0, 1)
    engine.charmm_step(t, p)
    e, w, _, _ = engine.fetch_energies()
    f = engine.fetch_forces()
    flj, elj, wlj = oracle.lj(so, t_o, 9.0, exclude=True)
    fe, ee, we = oracle.ewald_real(so, t_o, 0.35, 9.0, mdg.ELECTRIC, exclude=True)
    assert rel(e[0], elj) <= E_TOL and rel(e[1], ee) <= E_TOL
    assert force_err_rms(f, flj + fe) <= F_TOL
    np.testing.assert_allclose(w, wlj + we, rtol=0, atol=1e-9 * np.abs(wlj + we).max())


def test_imported_reference_table(engine, oracle, mdg):
    """A reference-layout table (exclusion-filtered) fed
    through mdg_nlist_import: the kernels see exactly that pair set."""
    s = mdg.water_box(216, 18.6, 3, "charmm")
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 8.0).filtered(s.molecule)
    engine.upload_system(s)
    t = engine.import_table(t_o.nnvlst, t_o.offset, t_o.indices, 8.0)
    np.testing.assert_array_equal(t.pairs(), t_o.pairs())
    fo, eo, _ = oracle.ewald_real(so, t_o, 0.35, 8.0)
    g = engine.ewald_real_forces(t, mdg.EwaldRealParams(0.35, 8.0))
    assert rel(g.energy, eo) <= E_TOL
    assert force_err_rms(g.forces, fo) <= F_TOL


def test_halgren_reduced_sites(engine, oracle, mdg):
    """Config-1 vdW: Halgren on H-reduced sites (factor 0.91), forces chain-ruled
    onto atoms; oracle = reference kernel on host-reduced coordinates."""
    s = mdg.water_box(1000, 31.04, 2, "amoeba")
    xr, yr, zr = oracle.reduce_sites(to_oracle_system(s), s.hred_parent, s.hred_factor)
    hx, hy, hz = mdg.reduce_sites_host(s)
    assert np.array_equal(xr, hx) and np.array_equal(yr, hy) and np.array_equal(zr, hz)
    so = to_oracle_system(s)
    so.x, so.y, so.z = xr, yr, zr
    t_o = oracle.build_table(so, 11.0)
    fred, eo, wo = oracle.halgren(so, t_o, 9.0, exclude=True)
    fo = oracle.reduce_forces(s.hred_parent, s.hred_factor, fred)
    engine.upload_system(s)
    t = engine.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
    np.testing.assert_array_equal(t.pairs(), t_o.pairs())  # device reduction is bit-exact
    g = engine.halgren_forces(t, mdg.HalgrenParams(9.0), exclude=True)
    assert rel(g.energy, eo) <= E_TOL
    assert force_err_rms(g.forces, fo) <= F_TOL


# ------------------------------------------------------------------ polarization
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_reference_fields(engine, oracle, mdg, seed):
    """proj/tests/test_polar.cpp:173-207: T mat-vec and charge field (alpha = 0)."""
    s = uniform(oracle, 260, 12.0, seed)
    t_o = oracle.build_table(s, 3.4)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.4)
    mu = oracle.random_dipoles(s.n, seed + 100)
    eo = oracle.tmatvec_thole(s, t_o, 3.0, 0.39, mu)
    st = mdg.PolarizationState(mu[:, 0], mu[:, 1], mu[:, 2], 0.39)
    g = engine.dipole_field_matvec(t, st, mdg.PolarParams(3.0, 0.39)).field
    assert force_err_max(g, eo) <= 1e-9
    eo = oracle.perm_field_thole(s, t_o, 3.0, 0.39)
    g = engine.permanent_field(t, mdg.PolarParams(3.0, 0.39)).field
    assert force_err_max(g, eo) <= 1e-9


def test_hand_fields(engine, oracle, mdg):
    """proj/tests/test_polar.cpp:117-171"""
    from oracle.oracle import System
    one = np.ones(2)
    s = System((10.0,) * 3, np.array([2.0, 2.0]), np.array([2.0, 2.0]), np.array([2.0, 4.0]),
               np.array([-3.0, 3.0]), one, one, one, one, one)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.0)
    st = mdg.PolarizationState(np.zeros(2), np.zeros(2), np.array([0.0, 1.0]), 1e9)
    f = engine.dipole_field_matvec(t, st, mdg.PolarParams(3.0, 1e9)).field
    assert f[0] == pytest.approx([0, 0, 0.25], abs=1e-12)
    st = mdg.PolarizationState(np.array([0.0, 1.0]), np.zeros(2), np.zeros(2), 1e9)
    f = engine.dipole_field_matvec(t, st, mdg.PolarParams(3.0, 1e9)).field
    assert f[0] == pytest.approx([-0.125, 0, 0], abs=1e-12)
    f = engine.permanent_field(t, mdg.PolarParams(3.0, 1e9)).field
    assert f[0][2] == pytest.approx(-0.75, abs=1e-12) and f[1][2] == pytest.approx(-0.75, abs=1e-12)


def test_jacobi_matches_oracle(engine, oracle, mdg):
    """proj/tests/test_polar.cpp:298-376 (converging small systems)."""
    for n in (6, 15):
        s = uniform(oracle, n, 9.0, 21)
        t_o = oracle.build_table(s, 3.0)
        mu_o, _ = oracle.jacobi(s, t_o, 3.0, 0.39, 1e-12, 500)
        engine.upload_system(s)
        t = engine.build_neighbor_table(3.0)
        st = engine.jacobi_polarization_solve(t, mdg.PolarParams(3.0, 0.39), 1e-12, 500)
        assert np.max(np.abs(st.mu - mu_o)) <= 1e-10 * max(1.0, np.abs(mu_o).max())


def test_jacobi_nonconvergence(engine, oracle, mdg):
    """proj/tests/test_polar.cpp:378-389"""
    s = uniform(oracle, 30, 9.0, 13)
    engine.upload_system(s)
    t = engine.build_neighbor_table(3.0)
    with pytest.raises(mdg.ConvergenceError) as ei:
        engine.jacobi_polarization_solve(t, mdg.PolarParams(3.0, 0.39), 1e-300, 2)
    assert ei.value.last_residual > 0


def amoeba_small(mdg, n_mol=1000, box=31.04, seed=4):
    return mdg.water_box(n_mol, box, seed, "amoeba")


def test_ewald_tmatvec_and_field(engine, oracle, mdg):
    """Ewald + Thole T and q/mu/Theta field (extensions) vs the oracle."""
    s = amoeba_small(mdg)
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 9.0)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.0)
    mu = oracle.random_dipoles(s.n_sites, 7, 0.05)
    eo = oracle.tmatvec_ewald(so, t_o, 0.5446, 7.0, 0.39, mu)
    st = mdg.PolarizationState(mu[:, 0], mu[:, 1], mu[:, 2], 0.39)
    g = engine.dipole_field_matvec(t, st, mdg.PolarParams(7.0, 0.39), alpha=0.5446).field
    assert force_err_rms(g, eo) <= F_TOL
    eo = oracle.perm_field_ewald(so, t_o, 0.5446, 7.0, 0.39, exclude=True)
    g = engine.permanent_field(t, mdg.PolarParams(7.0, 0.39), alpha=0.5446, exclude=True).field
    assert force_err_rms(g, eo) <= F_TOL


def test_pcg_matches_oracle(engine, oracle, mdg):
    """Config-2 solver on a 3000-atom box: same iterations (+-1) and dipoles
    within the 1e-5 D tolerance."""
    s = amoeba_small(mdg)
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 9.0)
    ep = oracle.perm_field_ewald(so, t_o, 0.5446, 7.0, 0.39, exclude=True)
    mu_o, it_o, rms_o = oracle.pcg(so, t_o, 0.5446, 7.0, 0.39, ep, 1e-5, 100)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.0)
    st = engine.polar_solve_pcg(t, mdg.PolarParams(7.0, 0.39), alpha=0.5446, tol_debye=1e-5,
                                max_iter=100, exclude_perm=True)
    assert abs(st.iterations - it_o) <= 1
    d = np.sqrt(np.mean(np.sum((st.mu - mu_o) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-5
    # the fused field + T-precompute pass produced the same right-hand side
    assert force_err_rms(engine.fetch_perm_field(), ep) <= F_TOL


def test_cluster_matvec_pcg_matches_oracle_and_per_site(engine, oracle, mdg):
    """The opt-in cluster PCG (3-site clusters = water molecules in the
    molecule-keyed order, union rows, TMA-staged mat-vec): the oracle's
    iterations (+-1) and dipoles within 1e-5 D, and the per-site path's
    dipoles, field and energies to rounding, over two steps (the second
    reuses the unions)."""
    s = amoeba_small(mdg, 1000, 31.04, 9)
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 9.0)
    ep = oracle.perm_field_ewald(so, t_o, 0.5446, 7.0, 0.39, exclude=True)
    mu_o, it_o, _ = oracle.pcg(so, t_o, 0.5446, 7.0, 0.39, ep, 1e-5, 100)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.0)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1)
    res = {}
    try:
        for on in (False, True):
            engine.set_cluster_matvec(on)
            for _ in range(2):
                engine.amoeba_step(t, t, p)
                e, w, iters, rms = engine.fetch_energies()
                res[on] = (e, iters, engine.fetch_dipoles(), engine.fetch_perm_field(),
                           engine.fetch_forces())
    finally:
        engine.set_cluster_matvec(False)
    e1, it1, mu1, ep1, f1 = res[True]
    e0, it0, mu0, ep0, f0 = res[False]
    assert abs(it1 - it_o) <= 1 and it1 == it0
    assert np.sqrt(np.mean(np.sum((mu1 - mu_o) ** 2, 1))) * mdg.DEBYE < 1e-5
    np.testing.assert_allclose(mu1, mu0, rtol=0, atol=1e-10 * np.abs(mu0).max())
    np.testing.assert_allclose(ep1, ep0, rtol=0, atol=1e-12 * np.abs(ep0).max())
    assert rel(e1[2], e0[2]) <= 1e-10
    np.testing.assert_allclose(f1, f0, rtol=0, atol=1e-12 * np.abs(f0).max())


def test_cluster_halgren_matches_per_site_and_oracle(engine, oracle, mdg):
    """Halgren on 3-site clusters (the default) against the per-site half rows
    and the oracle: energy, forces and virial, over two steps (the second
    reuses the unions), with the H reduction and exclusions of the AMOEBA
    water fixture (molecules straddle the periodic boundary)."""
    s = amoeba_small(mdg, 1000, 31.04, 12)
    so = to_oracle_system(s)
    so.x, so.y, so.z = oracle.reduce_sites(so, s.hred_parent, s.hred_factor)
    fred, eo, wo = oracle.halgren(so, oracle.build_table(so, 11.0), 9.0, exclude=True)
    fo = oracle.reduce_forces(s.hred_parent, s.hred_factor, fred)
    engine.upload_system(s)
    tv = engine.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
    out = {}
    try:
        for on in (False, True):
            engine.set_cluster_halgren(on)
            for _ in range(2):
                out[on] = engine.halgren_forces(tv, mdg.HalgrenParams(9.0), exclude=True)
    finally:
        engine.set_cluster_halgren(True)
    a, b = out[True], out[False]
    assert rel(a.energy, b.energy) <= 1e-12
    np.testing.assert_allclose(a.forces, b.forces, rtol=0, atol=1e-12 * np.abs(b.forces).max())
    np.testing.assert_allclose(a.virial, b.virial, rtol=0, atol=1e-12 * np.abs(b.virial).max())
    assert rel(a.energy, eo) <= E_TOL
    assert force_err_rms(a.forces, fo) <= F_TOL


@pytest.mark.parametrize("seed", [3, 8])
def test_irregular_molecules_order_and_cluster_halgren(engine, oracle, mdg, seed):
    """Molecule-keyed site order and Halgren clusters with irregular
    molecules: random molecule ids (1-5 sites, not contiguous in the caller's
    order, sites far apart), n not a multiple of 3. Exclusions follow the
    molecules; the cluster kernel, the per-site half rows and the oracle
    agree, and caller-order results are unaffected by the re-ordering."""
    rng = np.random.default_rng(seed)
    s = uniform(oracle, 1000, 24.0, seed)
    s.molecule = rng.integers(0, 330, s.n).astype(np.int32)
    so = to_oracle_system(s)
    fo, eo, wo = oracle.halgren(so, oracle.build_table(so, 7.0), 6.0, exclude=True)
    engine.upload_system(s)
    engine.upload_topology(s.molecule)
    t = engine.build_neighbor_table(7.0)
    out = {}
    try:
        for on in (True, False):
            engine.set_cluster_halgren(on)
            out[on] = engine.halgren_forces(t, mdg.HalgrenParams(6.0), exclude=True)
    finally:
        engine.set_cluster_halgren(True)
    for g in out.values():
        assert rel(g.energy, eo) <= E_TOL
        assert force_err_rms(g.forces, fo) <= F_TOL
    np.testing.assert_allclose(out[True].forces, out[False].forces, rtol=0,
                               atol=1e-12 * np.abs(fo).max())
    np.testing.assert_array_equal(t.pairs(), oracle.brute_force_pairs(s, 7.0))


def test_mpole_matches_oracle(engine, oracle, mdg):
    """Real-space multipole energy/forces/torques/virial vs the T-tensor oracle."""
    s = amoeba_small(mdg, 343, 21.0, 5)
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 9.0)
    fo, to, eo, wo = oracle.mpole(so, t_o, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.0)
    f, tq, e, w = engine.mpole_forces(t, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
    assert rel(e, eo) <= E_TOL
    assert force_err_rms(f, fo) <= F_TOL
    assert force_err_rms(tq, to) <= F_TOL
    np.testing.assert_allclose(w, wo, rtol=0, atol=1e-9 * np.abs(wo).max())


def test_amoeba_step_composes(engine, oracle, mdg):
    """The fused config-1..4 step == its parts."""
    s = amoeba_small(mdg, 343, 21.0, 6)
    engine.upload_system(s)
    tv = engine.build_neighbor_table(10.0, list_id=1, sites=mdg.SITES_VDW)
    te = engine.build_neighbor_table(9.0, list_id=0)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1)
    engine.amoeba_step(tv, te, p)
    e, w, iters, rms = engine.fetch_energies()
    f = engine.fetch_forces()
    mu = engine.fetch_dipoles()
    hv = engine.halgren_forces(tv, mdg.HalgrenParams(9.0), exclude=True)
    fm, _, em, wm = engine.mpole_forces(te, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
    st = engine.polar_solve_pcg(te, mdg.PolarParams(7.0, 0.39), 0.5446, 1e-5, 100, True)
    # Halgren: the same rows, the same sums. Multipoles: the step walks the
    # 7 A pruned rows, the standalone call its own cut of the 9 A list --
    # the same pairs on different lanes, so the sum order differs
    assert e[0] == hv.energy and rel(e[1], em) <= 1e-12
    # partner forces arrive through atomics (default half-row mode): the sum
    # order, not the terms, can differ between the fused step and its parts
    np.testing.assert_allclose(f, hv.forces + fm, rtol=0, atol=1e-12 * np.abs(f).max())
    assert iters == st.iterations and rms < 1e-5
    assert np.array_equal(mu, st.mu)
    np.testing.assert_allclose(w, hv.virial + wm, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("polar_force", [False, True])
def test_registered_force_output(engine, mdg, polar_force):
    """mdg_set_force_output: the step DMAs its final forces into the
    registered page-locked block (early, beside the PCG, or at the end when
    polarization forces still add to them); fetch_forces on that block right
    after the step only waits, and any call in between falls back to a fresh
    copy -- same bits as the plain fetch either way."""
    s = amoeba_small(mdg, 343, 21.0, 6)
    engine.upload_system(s)
    tv = engine.build_neighbor_table(10.0, list_id=1, sites=mdg.SITES_VDW)
    te = engine.build_neighbor_table(9.0, list_id=0)
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR
    if polar_force:
        terms |= mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
    n = len(s.x)
    buf = mdg.host_array((3, n))
    engine.set_force_output(buf)
    try:
        for between in (False, True, False):
            buf[:] = np.nan
            engine.amoeba_step(tv, te, p)
            if between:
                engine.fetch_energies()
            f = engine.fetch_forces(out=buf)
            ref = engine.fetch_forces()
            assert np.array_equal(f, ref)
            assert np.isfinite(buf).all()
        with pytest.raises(mdg.ContractViolation):
            engine.set_force_output(np.zeros((3, n)))  # pageable: rejected
    finally:
        engine.set_force_output(None)
    engine.amoeba_step(tv, te, p)
    buf[:] = 0.0
    f = engine.fetch_forces(out=buf)  # unregistered: plain copy
    assert np.array_equal(f, engine.fetch_forces())


def test_half_rows_match_deterministic_full_rows(engine, mdg):
    """Default mode (each owned pair once, partner force/torque by atomics)
    against the deterministic full-row mode, and the latter bitwise
    reproducible run to run."""
    s = amoeba_small(mdg, 343, 21.0, 7)
    engine.upload_system(s)
    tv = engine.build_neighbor_table(10.0, list_id=1, sites=mdg.SITES_VDW)
    te = engine.build_neighbor_table(9.0, list_id=0)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1)
    out = {}
    for mode in (False, True, True):
        engine.set_deterministic(mode)
        engine.amoeba_step(tv, te, p)
        e, w, it, _ = engine.fetch_energies()
        f = engine.fetch_forces()
        _, tq, _, _ = engine.mpole_forces(te, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
        cp = mdg.CharmmParams(9.0, 0.35, mdg.ELECTRIC, 0, 1)
        engine.charmm_step(te, cp)
        fc = engine.fetch_forces()
        ec = engine.fetch_energies()[0]
        out.setdefault(mode, []).append((e, w, f, tq, fc, ec))
    engine.set_deterministic(False)
    (e0, w0, f0, t0, fc0, ec0), = out[False]
    (e1, w1, f1, t1, fc1, ec1), (e2, w2, f2, t2, fc2, ec2) = out[True]
    for a, b in ((f1, f2), (t1, t2), (fc1, fc2), (e1, e2), (w1, w2), (ec1, ec2)):
        assert np.array_equal(a, b)
    np.testing.assert_allclose(e0, e1, rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(ec0, ec1, rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(w0, w1, rtol=0, atol=1e-11 * np.abs(w1).max())
    for a, b in ((f0, f1), (t0, t1), (fc0, fc1)):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12 * np.abs(b).max())


def test_site_type_tables_match_per_site_parameters(engine, mdg, monkeypatch):
    """Water has two parameter tuples, so the pair bodies read j's vdW
    parameters, charge and Thole factor from the context's type tables (type
    in the high word of pos.w); with MDG_NO_VDW_TYPES=1 they gather j's
    per-site records. Same values, so the deterministic (full-row) results of
    every kernel are bitwise identical."""
    engine.set_deterministic(True)
    out = []
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1,
                         mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE)
    for flag in ("0", "1"):
        monkeypatch.setenv("MDG_NO_VDW_TYPES", flag)
        s = mdg.water_box(343, 21.72, 5, "amoeba")
        engine.upload_system(s)
        tv = engine.build_neighbor_table(10.0, list_id=1, sites=mdg.SITES_VDW)
        te = engine.build_neighbor_table(9.0, list_id=0)
        h = engine.halgren_forces(tv, mdg.HalgrenParams(9.0), exclude=True)
        engine.amoeba_step(tv, te, p)
        e, w, it, _ = engine.fetch_energies()
        f = engine.fetch_forces()
        pf, ptq, pe, _ = engine.polar_forces(te, mdg.PolarParams(7.0, 0.39), 0.5446, mdg.ELECTRIC)
        s = mdg.water_box(343, 21.72, 5, "charmm")
        engine.upload_system(s)
        t = engine.build_neighbor_table(10.0)
        engine.charmm_step(t, mdg.CharmmParams(9.0, 0.35, mdg.ELECTRIC, 0, 1))
        ec = engine.fetch_energies()[0]
        fc = engine.fetch_forces()
        out.append((h.energy, h.forces.copy(), e, w, it, f, pf, ptq, pe, ec, fc))
    engine.set_deterministic(False)
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("buffer", ["0.5", "0"])
def test_buffered_rows_follow_motion(engine, oracle, mdg, monkeypatch, buffer):
    """The kernels walk rows cut to cutoff + 0.5 A (MDG_PRUNE_BUFFER) from the
    11 A list; the cut is redone on the device once some site has moved more
    than 0.25 A. Moves of 0.2 A (no new cut) and then 0.45 A in total (new cut)
    from the build positions: LJ on the unchanged 11 A list still matches the
    oracle on a table built at the new positions, so no pair that came within
    the cutoff was dropped. Buffer 0: the plain (lazily sorted) 11 A rows."""
    monkeypatch.setenv("MDG_PRUNE_BUFFER", buffer)
    s = mdg.water_box(1000, 31.04, 11, "charmm")
    engine.upload_system(s)
    t = engine.build_neighbor_table(11.0)
    rng = np.random.default_rng(5)
    d = rng.normal(size=(s.n_sites, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    L = s.box[0]
    for step in (0.2, 0.45):
        x = np.mod(np.asarray(s.x) + step * d[:, 0], L)
        y = np.mod(np.asarray(s.y) + step * d[:, 1], L)
        z = np.mod(np.asarray(s.z) + step * d[:, 2], L)
        x[x >= L] = 0.0
        y[y >= L] = 0.0
        z[z >= L] = 0.0
        engine.upload_positions(x, y, z)
        so = to_oracle_system(s)
        so.x, so.y, so.z = x, y, z
        t_o = oracle.build_table(so, 11.0)
        fo, eo, _ = oracle.lj(so, t_o, 9.0, exclude=True)
        g = engine.lj_forces(t, mdg.LjParams(9.0), exclude=True)
        assert rel(g.energy, eo) <= E_TOL
        assert force_err_rms(g.forces, fo) <= F_TOL


@pytest.mark.parametrize("deterministic", [False, True])
def test_polar_forces_match_oracle(engine, oracle, mdg, deterministic):
    """Polarization forces/torques/virial at fixed dipoles (8(f)#1) vs the
    tensor oracle (itself pinned by finite differences, test_oracle.py)."""
    s = amoeba_small(mdg, 343, 21.0, 9)
    so = to_oracle_system(s)
    t_o = oracle.build_table(so, 9.0)
    ep = oracle.perm_field_ewald(so, t_o, 0.5446, 7.0, 0.39, exclude=True)
    mu, _, _ = oracle.pcg(so, t_o, 0.5446, 7.0, 0.39, ep, 1e-8, 200)
    fo, to, eo, wo = oracle.polar_forces(so, t_o, 0.5446, 7.0, 0.39, mu, mdg.ELECTRIC)
    engine.upload_system(s)
    engine.set_deterministic(deterministic)
    t = engine.build_neighbor_table(9.0)
    f, tq, e, w = engine.polar_forces(t, mdg.PolarParams(7.0, 0.39), 0.5446, mdg.ELECTRIC, mu=mu)
    engine.set_deterministic(False)
    assert rel(e, eo) <= E_TOL
    assert force_err_rms(f, fo) <= F_TOL
    assert force_err_rms(tq, to) <= F_TOL
    np.testing.assert_allclose(w, wo, rtol=0, atol=1e-9 * np.abs(wo).max())


def test_amoeba_step_with_polar_forces_composes(engine, mdg):
    """TERM_POLAR_FORCE adds exactly the polarization forces at the step's
    own converged dipoles (pruned-row kernel == full-list API)."""
    s = amoeba_small(mdg, 343, 21.0, 10)
    engine.upload_system(s)
    tv = engine.build_neighbor_table(10.0, list_id=1, sites=mdg.SITES_VDW)
    te = engine.build_neighbor_table(9.0, list_id=0)
    base = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, base)
    engine.amoeba_step(tv, te, p)
    f0 = engine.fetch_forces()
    _, w0, _, _ = engine.fetch_energies()
    p.terms = base | mdg.TERM_POLAR_FORCE
    engine.amoeba_step(tv, te, p)
    f1 = engine.fetch_forces()
    e1, w1, _, _ = engine.fetch_energies()
    mu = engine.fetch_dipoles()
    fp, _, _, wp = engine.polar_forces(te, mdg.PolarParams(7.0, 0.39), 0.5446, mdg.ELECTRIC, mu=mu)
    scale = np.abs(f1).max()
    np.testing.assert_allclose(f1 - f0, fp, rtol=0, atol=1e-10 * scale)
    np.testing.assert_allclose(w1 - w0, wp, rtol=0, atol=1e-9 * np.abs(wp).max())


def test_device_erfc_accuracy(mdg):
    """The kernels' erfc (exp(-x^2) times the fitted erfcx polynomial,
    tools/fit_erfcx.py) against scipy's erfc on [0, 8] (library fallback
    beyond 6): ~8 ulp plus the rounding of x^2 amplified by exp, 2 x^2 ulp
    (measured: 1.7e-15 at x = 0.94, 4.5e-15 at x = 6). The energy tolerance
    this feeds is 1e-9."""
    from scipy.special import erfc
    x = np.concatenate([np.linspace(0.0, 8.0, 200001), np.random.default_rng(3).uniform(0, 6, 100000)])
    y = mdg.mdvec.device_erfc(x)
    ref = erfc(x)
    m = ref > 0
    rel = np.abs(y[m] - ref[m]) / ref[m]
    assert np.all(rel <= (8.0 + 2.0 * x[m] ** 2) * 2.0 ** -52)


def test_pcg_device_loop_max_iter_and_profiled_loop(engine, oracle, mdg):
    """The device-side PCG loop (CUDA while graph) stops at max_iter with
    ConvergenceError, and the host-driven loop (used while profiling) takes
    the same steps."""
    s = amoeba_small(mdg, 343, 21.0, 11)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.0)
    pp = mdg.PolarParams(7.0, 0.39)
    with pytest.raises(mdg.ConvergenceError) as ei:
        engine.polar_solve_pcg(t, pp, 0.5446, 1e-12, 3, True)
    assert ei.value.last_residual > 0
    a = engine.polar_solve_pcg(t, pp, 0.5446, 1e-7, 100, True)
    engine.profile(True)
    b = engine.polar_solve_pcg(t, pp, 0.5446, 1e-7, 100, True)
    engine.profile(False)
    assert a.iterations == b.iterations
    np.testing.assert_allclose(a.mu, b.mu, rtol=0, atol=1e-13 * np.abs(a.mu).max())


def test_pcg_graph_follows_new_box(engine, mdg):
    """The captured PCG loop is keyed on everything it holds by value: a new
    system of the same size in a different box re-captures it (dipoles as
    from a fresh context)."""
    pp = mdg.PolarParams(7.0, 0.39)
    a = amoeba_small(mdg, 343, 21.0, 11)
    b = amoeba_small(mdg, 343, 23.5, 12)
    engine.upload_system(a)
    engine.polar_solve_pcg(engine.build_neighbor_table(9.0), pp, 0.5446, 1e-7, 100, True)
    engine.upload_system(b)
    got = engine.polar_solve_pcg(engine.build_neighbor_table(9.0), pp, 0.5446, 1e-7, 100, True)
    with mdg.Engine(b.n_sites) as e:
        e.upload_system(b)
        want = e.polar_solve_pcg(e.build_neighbor_table(9.0), pp, 0.5446, 1e-7, 100, True)
    assert got.iterations == want.iterations
    # a stale graph (old box) would be off at ~1e-3; the two contexts may walk
    # different rows (the reused one can be in its buffered-row bypass after
    # many rebuilds: nlist.cu kernel_rows), i.e. sum the same pairs on other
    # lanes
    np.testing.assert_allclose(got.mu, want.mu, rtol=0, atol=1e-10 * np.abs(want.mu).max())


def test_isolated_sites_no_pairs(engine, oracle, mdg):
    """Edge case: every list row empty (2x2x2 lattice at 20 A spacing). Pair
    kernels return exact zeros, the PCG starts converged (E = 0, so mu = 0),
    the fused step composes to zeros -- no NaN from 0/0 in the CG scalars."""
    s = oracle.generate_system("lattice", 8, (40.0, 40.0, 40.0), 3)
    engine.upload_system(s)
    engine.upload_multipoles(np.zeros((8, 3)), np.zeros((8, 6)))
    t = engine.build_neighbor_table(9.0)
    assert len(t.pairs()) == 0
    lj = engine.lj_forces(t, mdg.LjParams(9.0))
    assert lj.energy == 0.0 and not np.any(lj.forces)
    hv = engine.halgren_forces(t, mdg.HalgrenParams(9.0))
    assert hv.energy == 0.0 and not np.any(hv.forces)
    st = engine.polar_solve_pcg(t, mdg.PolarParams(7.0, 0.39), 0.5446, 1e-5, 100, True)
    assert np.isfinite(st.mu).all() and not np.any(st.mu)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1,
                         mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE)
    engine.amoeba_step(t, t, p)
    e, w, iters, rms = engine.fetch_energies()
    assert np.isfinite(e).all() and np.isfinite(w).all() and rms == 0.0
    f = engine.fetch_forces()
    assert np.isfinite(f).all() and not np.any(f)


@pytest.mark.parametrize("n", [1, 2])
def test_tiny_systems(mdg, oracle, n):
    """One and two sites (the reference's smallest systems): list, pair
    kernels, PCG and the fused step on a context sized exactly n."""
    from oracle.oracle import System
    x = np.array([1.0, 3.5])[:n]
    one = np.ones(n)
    s = System((10.0, 10.0, 10.0), x.copy(), one * 2.0, one * 2.0, np.array([0.4, -0.4])[:n],
               one * 3.0, one * 0.1, one * 3.2, one * 0.05, one * 1.1)
    with mdg.Engine(n) as e:
        e.upload_system(s)
        e.upload_multipoles(np.zeros((n, 3)), np.zeros((n, 6)))
        t = e.build_neighbor_table(4.5)
        assert len(t.pairs()) == n - 1
        t_o = oracle.build_table(s, 4.5)
        fo, eo, _ = oracle.lj(s, t_o, 4.0)
        g = e.lj_forces(t, mdg.LjParams(4.0))
        assert rel(g.energy, eo) <= E_TOL and force_err_rms(g.forces, fo) <= F_TOL
        p = mdg.AmoebaParams(4.0, 0.07, 0.12, 4.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1,
                             mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR |
                             mdg.TERM_POLAR_FORCE)
        e.amoeba_step(t, t, p)
        en, w, iters, rms = e.fetch_energies()
        f = e.fetch_forces()
        assert np.isfinite(en).all() and np.isfinite(f).all() and rms < 1e-5
        np.testing.assert_allclose(f.sum(0), 0.0, atol=1e-12 * (np.abs(f).max() + 1))


def test_rows_longer_than_sort_limit(engine, oracle, mdg):
    """Rows over 1024 slots are left unsorted; the half-row kernels then
    split pairs by index in their prologue. Same forces as the deterministic
    full rows and the oracle."""
    s = uniform(oracle, 3000, 20.0, 5, min_sep=0.5)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.5)
    lp = mdg.LjParams(9.5)
    half = engine.lj_forces(t, lp)
    engine.set_deterministic(True)
    try:
        full = engine.lj_forces(t, lp)
    finally:
        engine.set_deterministic(False)
    np.testing.assert_allclose(half.forces, full.forces, rtol=0,
                               atol=1e-11 * np.abs(full.forces).max())
    assert rel(half.energy, full.energy) < 1e-12
    fo, eo, _ = oracle.lj(s, oracle.build_table(s, 9.5), 9.5)
    assert rel(half.energy, eo) <= E_TOL
    assert force_err_rms(half.forces, fo) <= F_TOL


def test_cut_rows_513_to_1024_slots(engine, oracle, mdg):
    """Buffered cut rows of 513-1024 slots take the second (32-register) sort
    launch (nlist.cu): ~610-slot 9.5 A rows here. Half rows + atomics ==
    deterministic full rows == the oracle."""
    s = uniform(oracle, 3000, 26.0, 6, min_sep=0.5)
    engine.upload_system(s)
    t = engine.build_neighbor_table(11.0)
    lp = mdg.LjParams(9.0)
    half = engine.lj_forces(t, lp)
    engine.set_deterministic(True)
    try:
        full = engine.lj_forces(t, lp)
    finally:
        engine.set_deterministic(False)
    np.testing.assert_allclose(half.forces, full.forces, rtol=0,
                               atol=1e-11 * np.abs(full.forces).max())
    fo, eo, _ = oracle.lj(s, oracle.build_table(s, 11.0), 9.0)
    assert rel(half.energy, eo) <= E_TOL
    assert force_err_rms(half.forces, fo) <= F_TOL


def test_amoeba_step_one_shared_list(engine, oracle, mdg):
    """one list for both the vdW and the electrostatic terms. The
    step then runs its two chains on one stream (no unordered cuts of the
    same buffered rows); results == the parts."""
    s = amoeba_small(mdg, 343, 21.0, 6)
    engine.upload_system(s)
    te = engine.build_neighbor_table(10.0, list_id=0)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1)
    for _ in range(3):
        engine.amoeba_step(te, te, p)
        e, w, iters, rms = engine.fetch_energies()
        f = engine.fetch_forces()
        hv = engine.halgren_forces(te, mdg.HalgrenParams(9.0), exclude=True)
        fm, _, em, wm = engine.mpole_forces(te, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
        assert rel(e[0], hv.energy) <= 1e-12 and rel(e[1], em) <= 1e-12
        np.testing.assert_allclose(f, hv.forces + fm, rtol=0, atol=1e-12 * np.abs(f).max())
        assert rms < 1e-5


def test_config4_full_size_properties(mdg):
    """BASELINE config 4 at full size (999,999 atoms), through size-independent
    properties: the 9 A list's pair count equals a KD-tree count, pair forces
    sum to zero, the default (half-row, atomic) and deterministic (full-row)
    modes agree, the PCG converges in the oracle's iteration count range."""
    from scipy.spatial import cKDTree
    s = mdg.water_box(333333, 215.3, 1, "amoeba")
    n = s.n_sites
    with mdg.Engine(n) as e:
        e.upload_system(s)
        te = e.build_neighbor_table(9.0, list_id=0)
        tv = e.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
        # pair count of the atomic 9 A list vs a periodic KD-tree
        pos = np.stack([s.x, s.y, s.z], 1)
        tree = cKDTree(pos, boxsize=215.3)
        half = (tree.count_neighbors(tree, 9.0) - n) // 2
        assert e.table_size(te)[0] == half
        p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1,
                             mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE)
        out = []
        for det in (False, True):
            e.set_deterministic(det)
            e.amoeba_step(tv, te, p)
            en, w, it, rms = e.fetch_energies()
            out.append((en, w, it, rms, e.fetch_forces().copy(), e.fetch_torques().copy()))
        e.set_deterministic(False)
    (en0, w0, it0, rms0, f0, t0), (en1, w1, it1, rms1, f1, t1) = out
    frms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(f0.sum(0)).max() <= 1e-9 * frms * np.sqrt(n)
    assert np.abs(f0 - f1).max() <= 1e-8 * frms
    assert np.abs(t0 - t1).max() <= 1e-8 * np.sqrt(np.mean(t1 ** 2))
    np.testing.assert_allclose(en0[:3], en1[:3], rtol=1e-9)
    assert 6 <= it0 <= 12 and abs(it0 - it1) <= 1 and rms0 < 1e-5


def test_local_frames_match_oracle(engine, oracle, mdg):
    """Local multipole frames (8(f)#2): rotation to the global frame and the
    torque -> frame-atom forces vs oracle/frames.py (itself pinned by finite
    differences); the permanent field and PCG see the rotated multipoles."""
    from oracle import frames as fr
    s = amoeba_small(mdg, 343, 21.0, 12)
    so = to_oracle_system(s)
    frame, za, xa = fr.water_frames(s.molecule)
    dl, ql = np.asarray(s.dipole), np.asarray(s.quadrupole)  # taken as local values
    pos = np.stack([s.x, s.y, s.z], 1)
    so.dipole, so.quadrupole = fr.rotate(pos, s.box, frame, za, xa, dl, ql)
    t_o = oracle.build_table(so, 9.0)
    fo, to, eo, wo = oracle.mpole(so, t_o, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
    fo = fo + fr.torque_forces(pos, s.box, frame, za, xa, to)
    engine.upload_system(s)
    engine.upload_frames(frame, za, xa, dl, ql)
    t = engine.build_neighbor_table(9.0)
    f, tq, e, w = engine.mpole_forces(t, 0.5446, 7.0, mdg.ELECTRIC, exclude=True)
    assert rel(e, eo) <= E_TOL
    assert force_err_rms(tq, to) <= F_TOL
    assert force_err_rms(f, fo) <= F_TOL
    # the field / solve use the rotated multipoles too
    ep = oracle.perm_field_ewald(so, t_o, 0.5446, 7.0, 0.39, exclude=True)
    st = engine.polar_solve_pcg(t, mdg.PolarParams(7.0, 0.39), 0.5446, 1e-5, 100, True)
    assert force_err_rms(engine.fetch_perm_field(), ep) <= F_TOL
    mu_o, it_o, _ = oracle.pcg(so, t_o, 0.5446, 7.0, 0.39, ep, 1e-5, 100)
    assert abs(st.iterations - it_o) <= 1
    assert np.sqrt(np.mean(np.sum((st.mu - mu_o) ** 2, 1))) * mdg.DEBYE < 1e-5
    engine.upload_frames(None, None, None)


def _charged_molecules(oracle, n_mol=30, L=20.0, seed=3):
    s = oracle.generate_system("uniform", 3 * n_mol, (L, L, L), seed, 1.0)
    s.charge[:] = np.tile([-0.8, 0.4, 0.4], n_mol)
    s.molecule = (np.arange(3 * n_mol) // 3).astype(np.int32)
    return s


def test_pme_matches_direct_ewald_sum(engine, oracle, mdg):
    """Smooth PME (8(f)#3) vs the direct structure-factor sum (oracle/
    ewald_recip.py) at PME accuracy; self and excluded-pair terms exact."""
    from oracle import ewald_recip as er
    s = _charged_molecules(oracle)
    L = s.box[0]
    pos = np.stack([s.x, s.y, s.z], 1)
    q = np.asarray(s.charge)
    e_o, f_o, w_o = er.recip(pos, q, s.box, 0.5, kmax=(24, 24, 24), electric=mdg.ELECTRIC)
    ex_o, fx_o, wx_o = er.excluded_correction(pos, q, s.box, s.molecule, 0.5, mdg.ELECTRIC)
    engine.upload_system(s)
    f, e, w = engine.ewald_recip(0.5, (48, 48, 48), 6, mdg.ELECTRIC, True)
    assert e[0] == pytest.approx(e_o, rel=1e-6)
    assert e[1] == pytest.approx(er.self_energy(q, 0.5, mdg.ELECTRIC), rel=1e-12)
    assert e[2] == pytest.approx(ex_o, rel=1e-12)
    fref = f_o + fx_o
    assert force_err_max(f, fref) <= 2e-5
    np.testing.assert_allclose(w, w_o + wx_o, rtol=0, atol=1e-5 * np.abs(w_o).max())


def test_mpole_pme_matches_direct_ewald_sum(engine, mdg):
    """Smooth PME of the permanent multipoles (q, mu, Theta; 8(f)#3) vs the
    direct structure-factor sum (oracle/ewald_mpole.py): energy, forces and
    torques at PME accuracy; self and excluded-pair terms exact."""
    from oracle import ewald_mpole as em
    s = mdg.water_box(64, 12.4, 3, "amoeba")
    pos = np.stack([s.x, s.y, s.z], 1)
    q, mu, q6 = np.asarray(s.charge), np.asarray(s.dipole), np.asarray(s.quadrupole)
    a = 0.5446
    e_o, f_o, t_o = em.recip(pos, q, mu, q6, s.box, a, kmax=(12, 12, 12), electric=mdg.ELECTRIC)
    ex_o, fx_o, tx_o = em.excluded_correction(pos, q, mu, q6, s.box, s.molecule, a,
                                              mdg.ELECTRIC, pair=em.mpole_pair)
    engine.upload_system(s)
    # PME converges spectrally in grid and order (measured at this alpha:
    # 48^3 / order 8: 1e-8 energy, 9e-7 forces; 64^3 / order 10: 9e-12, 1.3e-9)
    f, t, e = engine.ewald_recip_mpole(a, (64, 64, 64), 10, mdg.ELECTRIC, True)
    assert e[0] == pytest.approx(e_o, rel=1e-9)
    assert e[1] == pytest.approx(em.self_energy(q, mu, q6, a, mdg.ELECTRIC), rel=1e-12)
    assert e[2] == pytest.approx(ex_o, rel=1e-10)
    assert force_err_max(f, f_o + fx_o) <= 1e-7
    assert force_err_max(t, t_o + tx_o) <= 1e-7
    f8, t8, e8 = engine.ewald_recip_mpole(a, (48, 48, 48), 8, mdg.ELECTRIC, True)
    assert force_err_max(f8, f_o + fx_o) <= 1e-5  # the coarser grid at PME accuracy


def test_full_mpole_ewald_is_alpha_independent(engine, mdg):
    """Real-space multipoles (device kernel) + multipole PME + self + excluded
    pairs: the same total energy, forces and torques for two splitting
    parameters (the real-space sum converged within the 6 A cutoff)."""
    s = mdg.water_box(64, 12.4, 4, "amoeba")
    engine.upload_system(s)
    t = engine.build_neighbor_table(6.0)
    out = []
    for a in (0.8, 0.9):
        fr, tr, er, _ = engine.mpole_forces(t, a, 6.0, mdg.ELECTRIC, exclude=True)
        fk, tk, ek = engine.ewald_recip_mpole(a, (96, 96, 96), 10, mdg.ELECTRIC, True)
        out.append((er + ek.sum(), fr + fk, tr + tk))
    (e1, f1, t1), (e2, f2, t2) = out
    assert e1 == pytest.approx(e2, rel=1e-8)
    assert force_err_max(f1, f2) <= 1e-7
    assert force_err_max(t1, t2) <= 1e-7


def _full_ewald_polar_oracle(oracle, s, alpha, cutoff, thole=0.39, kmax=(10, 10, 10)):
    """Exact (dense) solution of (alpha^-1 - T_real - T_recip - self) mu =
    E_real + E_recip + self - E_excluded(erf) on a small box."""
    from oracle import ewald_mpole as em
    so = to_oracle_system(s)
    t = oracle.build_table(so, cutoff)
    pos = np.stack([s.x, s.y, s.z], 1)
    n = s.n_sites
    e_full = (oracle.perm_field_ewald(so, t, alpha, cutoff, thole, exclude=True)
              + em.field_recip(pos, s.charge, s.dipole, s.quadrupole, s.box, alpha, kmax)
              - em.excluded_field_erf(pos, s.charge, s.dipole, s.quadrupole, s.box,
                                      s.molecule, alpha))
    T = np.zeros((3 * n, 3 * n))
    for k in range(3 * n):
        u = np.zeros(3 * n)
        u[k] = 1.0
        T[:, k] = oracle.tmatvec_ewald(so, t, alpha, cutoff, thole, u.reshape(n, 3)).reshape(-1)
    T += em.tmat_recip_dense(pos, s.box, alpha, kmax)
    A = np.diag(np.repeat(1.0 / np.asarray(s.polarizability), 3)) - T
    mu = np.linalg.solve(A, e_full.reshape(-1)).reshape(n, 3)
    return mu, e_full


def test_pcg_with_reciprocal_space_matches_dense_solve(engine, oracle, mdg):
    """8(f)#3: the PCG with the reciprocal-space + self field in its operator
    and right-hand side (one smooth-PME pass per iteration) == the dense
    solve of the full Ewald + Thole system (oracle/ewald_mpole.py)."""
    s = mdg.water_box(27, 10.2, 5, "amoeba")
    a = 0.5446
    mu_o, e_o = _full_ewald_polar_oracle(oracle, s, a, 5.0)
    engine.upload_system(s)
    t = engine.build_neighbor_table(5.0)
    engine.set_ewald_recip((40, 40, 40), 8)
    try:
        st = engine.polar_solve_pcg(t, mdg.PolarParams(5.0, 0.39), alpha=a, tol_debye=1e-9,
                                    max_iter=200, exclude_perm=True)
        ep = engine.fetch_perm_field()
    finally:
        engine.set_ewald_recip((0, 0, 0))
    assert force_err_max(ep, e_o) <= 1e-7
    d = np.sqrt(np.mean(np.sum((st.mu - mu_o) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-7


def test_amoeba_step_with_reciprocal_space(engine, oracle, mdg):
    """The AMOEBA step with mdg_set_ewald_recip: multipole energy / forces /
    torques include the reciprocal, self and excluded-pair terms; the
    polarization energy is -1/2 mu.E_full of the full-Ewald solution."""
    from oracle import ewald_mpole as em
    from oracle.oracle import FastPort
    s = mdg.water_box(27, 10.2, 6, "amoeba")
    a = 0.5446
    so = to_oracle_system(s)
    pos = np.stack([s.x, s.y, s.z], 1)
    t_o = oracle.build_table(so, 5.0)
    fp = FastPort()
    fm, tm, em_real = fp.mpole(so, t_o, a, 5.0, mdg.ELECTRIC, True)
    ek, fk, tk = em.recip(pos, s.charge, s.dipole, s.quadrupole, s.box, a, (10, 10, 10),
                          mdg.ELECTRIC)
    ex, fx, tx = em.excluded_correction(pos, s.charge, s.dipole, s.quadrupole, s.box,
                                        s.molecule, a, mdg.ELECTRIC, pair=em.mpole_pair)
    es = em.self_energy(s.charge, s.dipole, s.quadrupole, a, mdg.ELECTRIC)
    mu_o, e_o = _full_ewald_polar_oracle(oracle, s, a, 5.0)
    engine.upload_system(s)
    te = engine.build_neighbor_table(5.0, list_id=0)
    p = mdg.AmoebaParams(4.5, 0.07, 0.12, 5.0, a, mdg.ELECTRIC, 0.39, 1e-9, 200, 1,
                         mdg.TERM_MPOLE | mdg.TERM_POLAR)
    engine.set_ewald_recip((40, 40, 40), 8)
    try:
        engine.amoeba_step(te, te, p)
        e, w, it, rms = engine.fetch_energies()
        f, tq, mu = engine.fetch_forces(), engine.fetch_torques(), engine.fetch_dipoles()
    finally:
        engine.set_ewald_recip((0, 0, 0))
    # the terms cancel (|E| ~ 60 of |terms| ~ 2500): PME accuracy on the terms
    scale = abs(em_real) + abs(ek) + abs(es) + abs(ex)
    assert abs(e[1] - (em_real + ek + es + ex)) <= 1e-8 * scale
    assert force_err_max(f, fm + fk + fx) <= 1e-6
    assert force_err_max(tq, tm + tk + tx) <= 1e-6
    assert np.sqrt(np.mean(np.sum((mu - mu_o) ** 2, 1))) * mdg.DEBYE < 1e-7
    assert rel(e[2], -0.5 * mdg.ELECTRIC * float(np.sum(mu_o * e_o))) <= 1e-7


def test_polar_forces_with_reciprocal_space_by_fd(engine, oracle, mdg):
    """Multipole + polarization forces with reciprocal space (the permanent +
    induced set's PME pass after the solve) == -dE/dx of the oracle's full
    Ewald energy E_mpole + E_pol (dense solve re-done at every displaced
    geometry: the variational polarization energy)."""
    from oracle import ewald_mpole as em
    from oracle.oracle import FastPort
    s = mdg.water_box(27, 10.2, 7, "amoeba")
    a = 0.5446
    fp = FastPort()

    def energy(x):
        q = mdg.water_box(27, 10.2, 7, "amoeba")
        q.x, q.y, q.z = x[:, 0].copy(), x[:, 1].copy(), x[:, 2].copy()
        so = to_oracle_system(q)
        e_real = fp.mpole(so, oracle.build_table(so, 5.0), a, 5.0, mdg.ELECTRIC, True)[2]
        e_rec = em.recip(x, q.charge, q.dipole, q.quadrupole, q.box, a, (10, 10, 10),
                         mdg.ELECTRIC, energy_only=True)[0]
        e_ex = em.excluded_correction(x, q.charge, q.dipole, q.quadrupole, q.box, q.molecule,
                                      a, mdg.ELECTRIC, pair=em.mpole_pair)[0]
        mu, e_full = _full_ewald_polar_oracle(oracle, q, a, 5.0)
        return e_real + e_rec + e_ex - 0.5 * mdg.ELECTRIC * float(np.sum(mu * e_full))

    engine.upload_system(s)
    te = engine.build_neighbor_table(5.0, list_id=0)
    p = mdg.AmoebaParams(4.5, 0.07, 0.12, 5.0, a, mdg.ELECTRIC, 0.39, 1e-10, 300, 1,
                         mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE)
    engine.set_ewald_recip((48, 48, 48), 10)
    try:
        engine.amoeba_step(te, te, p)
        f = engine.fetch_forces()
    finally:
        engine.set_ewald_recip((0, 0, 0))
    x0 = np.stack([s.x, s.y, s.z], 1)
    h = 1e-4
    fmax = np.abs(f).max()
    for i, k in ((0, 0), (10, 1), (41, 2), (70, 0)):
        xp, xm = x0.copy(), x0.copy()
        xp[i, k] += h
        xm[i, k] -= h
        num = -(energy(xp) - energy(xm)) / (2 * h)
        assert abs(f[i, k] - num) <= 1e-6 * fmax, (i, k, f[i, k], num)


def test_full_ewald_is_alpha_independent(engine, oracle, mdg):
    """Real space (device kernel) + PME + self + excluded pairs: the same
    total energy and forces for two splitting parameters."""
    s = _charged_molecules(oracle, seed=4)
    engine.upload_system(s)
    t = engine.build_neighbor_table(9.9)
    tot = []
    for a in (0.5, 0.6):
        rs = engine.ewald_real_forces(t, mdg.EwaldRealParams(a, 9.9), exclude=True)
        f, e, w = engine.ewald_recip(a, (64, 64, 64), 8, 1.0, True)
        tot.append((rs.energy + e.sum(), rs.forces + f, np.abs(e).max()))
    # the terms are O(10) and nearly cancel: PME accuracy relative to them
    assert abs(tot[0][0] - tot[1][0]) <= 1e-6 * tot[0][2]
    assert force_err_max(tot[0][1], tot[1][1]) <= 2e-5


# ---------------------------------------------------------------- MD loop (8(f)#4)
def _md_water(mdg, n_mol=216, box=18.6, seed=2, temp=300.0):
    from oracle import md
    s = mdg.water_box(n_mol, box, seed, "charmm")
    n = s.n_sites
    mass = np.tile([15.999, 1.008, 1.008], n_mol)
    rng = np.random.default_rng(seed)
    kT = 0.0019872041 * temp
    vel = rng.normal(size=(n, 3)) * np.sqrt(kT * md.ACCEL / mass)[:, None]
    vel -= (mass[:, None] * vel).sum(0) / mass.sum()
    b, a = md.water_topology(n_mol)
    return s, mass, vel, b, a


def test_bonded_forces_match_oracle(engine, oracle, mdg):
    from oracle import md
    s, mass, vel, b, a = _md_water(mdg, 27, 9.4, 3)
    # distort the rigid fixture geometry (bonds and angles off their minima)
    rng = np.random.default_rng(8)
    for k in ("x", "y", "z"):
        getattr(s, k)[:] = np.mod(getattr(s, k) + rng.normal(0, 0.05, s.n_sites), 9.4)
    pos = np.stack([s.x, s.y, s.z], 1)
    eb, ea, fo = md.bonded(pos, s.box, b, 529.6, 0.9572, a, 34.05, np.deg2rad(104.52))
    engine.upload_system(s)
    engine.upload_bonded(b, 529.6, 0.9572, a, 34.05, np.deg2rad(104.52))
    f, e = engine.bonded_forces()
    assert e[0] == pytest.approx(eb, rel=1e-12) and e[1] == pytest.approx(ea, rel=1e-12)
    assert force_err_max(f, fo) <= 1e-12


def test_md_trajectory_matches_oracle(engine, oracle, mdg, monkeypatch):
    """20 velocity-Verlet steps of flexible CHARMM-style water on the device
    against the numpy integrator driven by the oracle's forces (the sites
    re-sorted on the device at each of the two list rebuilds)."""
    from oracle import md
    monkeypatch.setenv("MDG_RESORT", "1")
    s, mass, vel, b, a = _md_water(mdg)
    so = to_oracle_system(s)
    bond_args = (b, 529.6, 0.9572, a, 34.05, np.deg2rad(104.52))
    t_o = oracle.build_table(so, 9.3)

    def force_fn(pos):
        q = so.copy()
        q.x[:], q.y[:], q.z[:] = pos[:, 0], pos[:, 1], pos[:, 2]
        t = oracle.build_table(q, 9.3)
        f1, e1, _ = oracle.lj(q, t, 8.0, shift=True, exclude=True)
        f2, e2, _ = oracle.ewald_real(q, t, 0.45, 8.0, mdg.ELECTRIC, exclude=True)
        eb, ea, f3 = md.bonded(pos, so.box, *bond_args)
        return f1 + f2 + f3, e1 + e2 + eb + ea

    pos0 = np.stack([s.x, s.y, s.z], 1)
    p_o, v_o, ek_o, ep_o = md.velocity_verlet(pos0, vel, mass, so.box, force_fn, 0.5, 20)
    engine.upload_system(s)
    engine.upload_bonded(*bond_args)
    engine.upload_velocities(vel, mass)
    p = mdg.MDParams(0, 20, 0.5, 10, 0, 1, 9.3, 0.0, 1)
    ek, ep = engine.md_run(p, charmm=mdg.CharmmParams(8.0, 0.45, mdg.ELECTRIC, 1, 1))
    pos = engine.fetch_positions()
    d = pos - p_o
    d -= np.asarray(so.box) * np.rint(d / np.asarray(so.box))
    assert np.abs(d).max() <= 1e-9
    assert np.abs(engine.fetch_velocities() - v_o).max() <= 1e-9 * np.abs(v_o).max()
    np.testing.assert_allclose(ek, ek_o, rtol=1e-9)
    np.testing.assert_allclose(ep, ep_o, rtol=1e-9)


def test_resort_keeps_every_result(engine, oracle, mdg):
    """mdg_resort (device spatial re-sort) on a system with
    topology, H reduction, local frames, bonds/angles and velocities: the
    caller-order results of the AMOEBA step (energies, forces, torques,
    dipoles), the bonded forces and the coordinates / velocities are the same
    after the re-sort (to FP64 summation order), including after the sites
    were moved far from their cells."""
    from oracle import frames as fr
    s = mdg.water_box(512, 24.8, 3, "amoeba")
    frame, za, xa = fr.water_frames(s.molecule)
    n_mol = s.n_sites // 3
    bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2),
                      (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
    angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3,
                       np.arange(n_mol) * 3 + 2], 1)
    mass = np.tile([15.999, 1.008, 1.008], n_mol)
    vel = np.random.default_rng(4).normal(size=(s.n_sites, 3)) * 0.005
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-6, 100, 1,
                         mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE)
    engine.upload_system(s)
    engine.upload_frames(frame, za, xa, np.asarray(s.dipole), np.asarray(s.quadrupole))
    engine.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
    engine.upload_velocities(vel, mass)
    # move every molecule to another molecule's place: the stored order no
    # longer follows space
    perm = np.random.default_rng(5).permutation(n_mol)
    xyz = np.stack([s.x, s.y, s.z], 1).reshape(n_mol, 3, 3)[perm].reshape(-1, 3)
    engine.upload_positions(xyz[:, 0], xyz[:, 1], xyz[:, 2])

    def results():
        tv = engine.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
        te = engine.build_neighbor_table(9.0, list_id=0)
        engine.amoeba_step(tv, te, p)
        e, w, it, rms = engine.fetch_energies()
        fb, eb = engine.bonded_forces()
        return (e, w, engine.fetch_forces(), engine.fetch_torques(), engine.fetch_dipoles(),
                fb, eb, engine.fetch_positions(), engine.fetch_velocities())

    before = results()
    engine.resort()
    after = results()
    e0, w0, f0, t0, mu0, fb0, eb0, x0, v0 = before
    e1, w1, f1, t1, mu1, fb1, eb1, x1, v1 = after
    np.testing.assert_allclose(e1[:3], e0[:3], rtol=1e-11)
    np.testing.assert_allclose(w1, w0, rtol=1e-10, atol=1e-10 * np.abs(w0).max())
    assert force_err_max(f1, f0) <= 1e-11
    assert force_err_max(t1, t0) <= 1e-11
    assert np.abs(mu1 - mu0).max() <= 1e-10 * np.abs(mu0).max()
    assert force_err_max(fb1, fb0) <= 1e-12 and np.allclose(eb1, eb0, rtol=1e-12)
    assert np.array_equal(x1, x0) and np.array_equal(v1, v0)


def test_md_energy_conservation(engine, mdg):
    """NVE: 2,000 steps of 0.25 fs -- the total energy stays flat."""
    s, mass, vel, b, a = _md_water(mdg, seed=4)
    engine.upload_system(s)
    engine.upload_bonded(b, 529.6, 0.9572, a, 34.05, np.deg2rad(104.52))
    engine.upload_velocities(vel, mass)
    p = mdg.MDParams(0, 2000, 0.25, 20, 0, 1, 9.3, 0.0, 1)
    ek, ep = engine.md_run(p, charmm=mdg.CharmmParams(8.0, 0.45, mdg.ELECTRIC, 1, 1))
    et = ek + ep
    assert np.all(np.isfinite(et))
    assert (et.max() - et.min()) <= 2e-3 * ek.mean()


@pytest.mark.parametrize("buffered", [False, True])
def test_outdated_list_is_reported(engine, oracle, mdg, monkeypatch, buffered):
    """A list walked after its sites moved more than half its skin (list
    cutoff - kernel cutoff, less the row buffer on the buffered path) would
    miss pairs: the next read of the results raises ContractViolation, and a
    rebuild clears it. Motion within the bound is accepted."""
    monkeypatch.setenv("MDG_PRUNE_MIN_SITES", "0" if buffered else "100000000")
    s = mdg.water_box(1000, 31.04, 1, "amoeba")
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1,
                         mdg.TERM_VDW | mdg.TERM_MPOLE)
    engine.upload_system(s)
    te = engine.build_neighbor_table(9.0, list_id=0)
    tv = engine.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
    engine.amoeba_step(tv, te, p)
    engine.fetch_energies()
    L = 31.04
    rng = np.random.default_rng(1)
    # within the bound: 0.3 A (the buffered bound is (9 - 7.5) / 2 = 0.75 A)
    small = [np.mod(np.asarray(getattr(s, k)) + rng.uniform(-0.3, 0.3, s.n_sites) / np.sqrt(3), L)
             for k in ("x", "y", "z")]
    engine.upload_positions(*small)
    engine.amoeba_step(tv, te, p)
    engine.fetch_energies()
    # past it: one site moved 1.6 A
    big = [a.copy() for a in small]
    big[0][5] = np.mod(big[0][5] + 1.6, L)
    engine.upload_positions(*big)
    engine.amoeba_step(tv, te, p)
    with pytest.raises(mdg.ContractViolation):
        engine.fetch_energies()
    te = engine.build_neighbor_table(9.0, list_id=0)
    tv = engine.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
    engine.amoeba_step(tv, te, p)
    engine.fetch_energies()
