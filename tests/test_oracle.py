"""CPU: pin the oracle (oracle/mdo.c) before trusting it.

1. Known-answer vectors carried over from the reference's own tests
   (proj/tests/test_pbc.cpp, test_kernels.cpp, test_polar.cpp).
2. Bit-for-bit / tolerance agreement with the unmodified reference library
   (oracle/_ref, built here from /root/reference) -- skipped where absent;
   tests/test_golden.py covers the same ground from committed fixtures.
3. Limit and property tests for the extensions the reference lacks
   (SURVEY 8(c) gap ledger): alpha -> 0, multipoles -> charges, finite
   differences, torques by finite rotation, dense solves, T symmetry.
"""
import numpy as np
import pytest

from oracle.oracle import OracleError, System


def two_site(a, b, box=10.0, **kw):
    one = np.ones(2)
    s = System((box, box, box), np.array([a, b]), np.array([5.0, 5.0]), np.array([5.0, 5.0]),
               np.array([1.0, 1.0]), one.copy(), one.copy(), one.copy(), one.copy(), one.copy())
    for k, v in kw.items():
        setattr(s, k, v)
    return s


# ------------------------------------------------------------------- KATs
def test_minimum_image_examples(oracle):
    """proj/tests/test_pbc.cpp:21-46"""
    w = lambda d: oracle.wrap1(d, 10.0)  # noqa: E731
    assert w(7) == -3.0 and w(-6) == 4.0 and w(5) == -5.0 and w(-5) == -5.0
    assert oracle.minimum_image((2.5, -7.5, 9.0), (10, 10, 10)) == (2.5, 2.5, -1.0)


def test_minimum_image_range(oracle):
    """proj/tests/test_pbc.cpp:48-62"""
    rng = np.random.default_rng(11)
    for L in (7.5, 10.0, 3.25):
        for d in rng.uniform(-60, 60, 2000):
            t = oracle.wrap1(d, L)
            assert -L / 2 <= t < L / 2
            assert oracle.wrap1(t, L) == t  # idempotent (test_pbc.cpp:64-77)


def test_lj_kat(oracle):
    """proj/tests/test_kernels.cpp:72-75: exact values at r^2 = 4."""
    s = two_site(1.0, 3.0)
    t = oracle.build_table(s, 3.0)
    f, e, _ = oracle.lj(s, t, 3.0)
    assert e == -0.0615234375
    assert f[0, 0] == -0.0908203125 * -2.0


def test_ewald_kat(oracle):
    """proj/tests/test_kernels.cpp:86-94"""
    s = two_site(1.0, 4.0)
    t = oracle.build_table(s, 3.5)
    f, e, _ = oracle.ewald_real(s, t, 0.4, 3.5)
    assert e == pytest.approx(0.02989534059012154, rel=1e-15)
    assert -f[0, 0] / 3.0 == pytest.approx(0.015203675487948578, rel=1e-15)
    s.charge[:] = [3.0, -1.5]
    s.x[:] = [1.0, 3.0]
    f, e, _ = oracle.ewald_real(s, t, 0.0, 3.5)
    assert e == pytest.approx(-4.5 / 2.0, rel=1e-15)
    assert -f[0, 0] / 2.0 == pytest.approx(-4.5 / 8.0, rel=1e-15)


def test_halgren_kat(oracle):
    """proj/tests/test_polar.cpp:52-67: u(1.5), dU/drho(1.5), dU/drho(1)."""
    s = two_site(1.0, 2.5)  # r = 1.5, r0 = 1, eps = 1
    t = oracle.build_table(s, 3.0)
    f, e, _ = oracle.halgren(s, t, 3.0)
    assert e == pytest.approx(-0.13214440848300467, rel=1e-14)
    # F_i = fs d, fs = -dudrho / (r0 r), d = -1.5
    dudrho = f[0, 0] / 1.5 * 1.5
    assert dudrho == pytest.approx(0.5685775350898349, rel=1e-13)
    s = two_site(1.0, 2.0)
    f, e, _ = oracle.halgren(s, oracle.build_table(s, 3.0), 3.0)
    assert e == pytest.approx(-1.0, rel=1e-15)
    assert f[0, 0] == pytest.approx(0.29205607476635514, rel=1e-13)


def test_thole_kat(oracle):
    """proj/tests/test_polar.cpp:92-95: l3, l5 at r = 2, alpha = 1, a = 0.39."""
    s = two_site(1.0, 3.0)
    s.charge[:] = [0.0, 1.0]
    t = oracle.build_table(s, 3.0)
    e = oracle.perm_field_thole(s, t, 3.0, 0.39)
    l3 = -e[0, 0] * 4.0  # E_0 = l3 q_1 d / r^3, d = -2
    assert l3 == pytest.approx(0.9558428315803071, rel=1e-15)
    mu = np.array([[0, 0, 0], [1.0, 0, 0]])
    e = oracle.tmatvec_thole(s, t, 3.0, 0.39, mu)
    # axial: E_x = (3 l5 - l3) / 8
    l5 = (8 * e[0, 0] + l3) / 3
    assert l5 == pytest.approx(0.8180724661108654, rel=1e-14)


def test_hand_fields(oracle):
    """proj/tests/test_polar.cpp:117-171"""
    one = np.ones(2)
    s = System((10.0,) * 3, np.array([2.0, 2.0]), np.array([2.0, 2.0]), np.array([2.0, 4.0]),
               np.array([-3.0, 3.0]), one, one, one, one, one)
    t = oracle.build_table(s, 3.0)
    f = oracle.tmatvec_thole(s, t, 3.0, 1e9, np.array([[0, 0, 0], [0, 0, 1.0]]))
    assert f[0] == pytest.approx([0, 0, 0.25], abs=1e-12)
    f = oracle.tmatvec_thole(s, t, 3.0, 1e9, np.array([[0, 0, 0], [1.0, 0, 0]]))
    assert f[0] == pytest.approx([-0.125, 0, 0], abs=1e-12)
    f = oracle.perm_field_thole(s, t, 3.0, 1e9)
    assert f[0, 2] == pytest.approx(-0.75, abs=1e-12) and f[1, 2] == pytest.approx(-0.75, abs=1e-12)


def test_table_invariants_and_brute_force(oracle):
    """proj/tests/test_neighbors.cpp:137-148, 186-204"""
    for seed in (1, 2, 3):
        for n in (32, 150, 700):
            s = oracle.generate_system("uniform", n, (14, 14, 14), seed)
            t = oracle.build_table(s, 3.4)
            np.testing.assert_array_equal(t.pairs(), oracle.brute_force_pairs(s, 3.4))
            assert np.all(t.offset % 16 == 0)
    s = oracle.generate_system("uniform", 200, (11, 11, 11), 5)
    a, b = oracle.build_table(s, 3.0), oracle.build_table(s, 3.0, 32)
    np.testing.assert_array_equal(a.nnvlst, b.nnvlst)
    assert np.all(b.nvloop16 == a.nvloop16 + 32)
    np.testing.assert_array_equal(a.pairs(), b.pairs())


def test_capacity_and_contracts(oracle):
    """proj/tests/test_neighbors.cpp:214-230"""
    s = oracle.generate_system("uniform", 6000, (9, 9, 9), 8, 0.05)
    with pytest.raises(OracleError) as ei:
        oracle.build_table(s, 4.4)
    assert ei.value.code == 2
    s = oracle.generate_system("uniform", 20, (10, 10, 10), 1)
    for bad in (0.0, 6.1):
        with pytest.raises(OracleError) as ei:
            oracle.build_table(s, bad)
        assert ei.value.code == 1


# ------------------------------------------------- against the real reference
def test_generator_bit_exact_vs_reference(oracle, ref):
    for kind in ("uniform", "lattice"):
        for seed in (1, 2, 3):
            a = oracle.generate_system(kind, 300, (12, 13, 14), seed)
            b = ref.generate_system(kind, 300, (12, 13, 14), seed)
            for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0",
                      "hal_epsilon", "polarizability"):
                assert np.array_equal(getattr(a, k), getattr(b, k)), (kind, seed, k)
    assert np.array_equal(oracle.random_dipoles(50, 3), ref.random_dipoles(50, 3))


@pytest.mark.parametrize("seed", [9, 10, 11])
def test_table_identical_to_reference(oracle, ref, seed):
    """Slot for slot, both reference builders (test_neighbors.cpp:150-169)."""
    s = oracle.generate_system("uniform", 400, (13, 13, 13), seed)
    h = ref.handle(s)
    mine = oracle.build_table(s, 3.0)
    for vec in (True, False):
        r = h.build_table(3.0, vec=vec)
        for k in ("nnvlst", "nvloop8", "nvloop16", "offset", "indices", "scale"):
            assert np.array_equal(getattr(mine, k), getattr(r, k)), k
    np.testing.assert_array_equal(mine.pairs(), h.brute_force_pairs(3.0))


@pytest.mark.parametrize("seed", [1, 4, 7])
def test_kernels_match_reference(oracle, ref, seed):
    s = oracle.generate_system("uniform", 333, (12, 12, 12), seed)
    h = ref.handle(s)
    rt = h.build_table(3.7)
    t = oracle.build_table(s, 3.7)
    for vec in (False, True):
        f, e = h.forces("lj", 3.0, vec=vec)
        fo, eo, _ = oracle.lj(s, t, 3.0)
        assert abs(e - eo) <= 1e-12 * abs(e) and np.abs(f - fo).max() <= 1e-12 * np.abs(f).max()
        f, e = h.forces("ewald_real", 3.7, 0.4, vec=vec)
        fo, eo, _ = oracle.ewald_real(s, t, 0.4, 3.7)
        assert abs(e - eo) <= 1e-12 * abs(e) and np.abs(f - fo).max() <= 1e-12 * np.abs(f).max()
        f, e = h.forces("halgren", 3.0, 0.07, 0.12, vec=vec)
        fo, eo, _ = oracle.halgren(s, t, 3.0)
        assert abs(e - eo) <= 1e-12 * abs(e) and np.abs(f - fo).max() <= 1e-12 * np.abs(f).max()
        mu = oracle.random_dipoles(s.n, seed + 100)
        a = h.field("tmatxb", 3.0, 0.39, mu, vec=vec)
        assert np.abs(a - oracle.tmatvec_thole(s, t, 3.0, 0.39, mu)).max() <= 1e-12 * np.abs(a).max()
        a = h.field("perm", 3.0, 0.39, vec=vec)
        assert np.abs(a - oracle.perm_field_thole(s, t, 3.0, 0.39)).max() <= 1e-12 * np.abs(a).max()
    assert rt.total == t.indices.shape[0] if hasattr(rt, "total") else True


def test_jacobi_matches_reference(oracle, ref):
    for n in (6, 15):
        s = oracle.generate_system("uniform", n, (9, 9, 9), 21)
        h = ref.handle(s)
        h.build_table(3.0)
        mr = h.jacobi(3.0, 0.39, 1e-12, 500)
        mo, _ = oracle.jacobi(s, oracle.build_table(s, 3.0), 3.0, 0.39, 1e-12, 500)
        assert np.abs(mr - mo).max() <= 1e-12
    s = oracle.generate_system("uniform", 30, (9, 9, 9), 13)
    with pytest.raises(OracleError) as ei:
        oracle.jacobi(s, oracle.build_table(s, 3.0), 3.0, 0.39, 1e-300, 2)
    assert ei.value.code == 4 and ei.value.last_residual > 0


def test_exclusion_filter_equals_reference_on_filtered_table(oracle, ref):
    """exclusions = reference kernels on a segment-filtered table."""
    s = oracle.generate_system("lattice", 300, (15, 15, 15), 3)
    s.molecule = (np.arange(s.n) // 3).astype(np.int32)
    t = oracle.build_table(s, 4.0)
    tf = t.filtered(s.molecule)
    h = ref.handle(s)
    h.set_table(tf)
    f, e = h.forces("ewald_real", 4.0, 0.35, vec=False)
    fo, eo, _ = oracle.ewald_real(s, t, 0.35, 4.0, exclude=True)
    assert abs(e - eo) <= 1e-12 * abs(e) and np.abs(f - fo).max() <= 1e-12 * np.abs(f).max()


# ------------------------------------------------------- properties / extensions
def fd_forces(energy_fn, s, h=1e-6):
    out = np.zeros((s.n, 3))
    for i in range(s.n):
        for a, k in enumerate("xyz"):
            arr = getattr(s, k)
            saved = arr[i]
            arr[i] = saved + h
            up = energy_fn(s)
            arr[i] = saved - h
            dn = energy_fn(s)
            arr[i] = saved
            out[i, a] = -(up - dn) / (2 * h)
    return out


def test_fd_forces_lj_ewald_halgren(oracle):
    """proj/tests/test_kernels.cpp:197-246, test_polar.cpp:209-239"""
    s = oracle.generate_system("uniform", 10, (8, 8, 8), 31)
    cases = [lambda s, t: oracle.lj(s, t, 3.0, shift=True),
             lambda s, t: oracle.ewald_real(s, t, 0.5, 3.0),
             lambda s, t: oracle.halgren(s, t, 3.0)]
    for fn in cases:
        f = fn(s, oracle.build_table(s, 3.4))[0]
        num = fd_forces(lambda q: fn(q, oracle.build_table(q, 3.4))[1], s)
        assert np.all(np.abs(num - f) <= 1e-5 * np.maximum(1.0, np.abs(f)))


def test_momentum_and_virial(oracle):
    """Sum F = 0 (acceptance.cpp:256-299); virial trace = -dE/d(eps) under
    affine scaling of positions and box (no pair crosses the cutoff)."""
    s = oracle.generate_system("uniform", 200, (12, 12, 12), 3)
    t = oracle.build_table(s, 3.4)
    f, e, w = oracle.lj(s, t, 3.0)
    assert np.abs(f.sum(0)).max() <= 1e-9 * np.abs(f).max()
    assert np.allclose(w, w.T, rtol=1e-12, atol=1e-12 * np.abs(w).max())

    def energy_scaled(eps):
        q = s.copy()
        q.box = tuple(b * (1 + eps) for b in s.box)
        for k in "xyz":
            setattr(q, k, getattr(s, k) * (1 + eps))
        return oracle.lj(q, t, 3.0 * 1.0)[1]  # same table (pair set fixed)
    h = 1e-7
    dEde = (energy_scaled(h) - energy_scaled(-h)) / (2 * h)
    # pairs near the cutoff would make this ill-posed; the uniform system has a gap
    assert np.trace(w) == pytest.approx(-dEde, rel=1e-5)


def test_ewald_field_and_T_reduce_to_reference_at_alpha0(oracle):
    s = oracle.generate_system("uniform", 150, (11, 11, 11), 4)
    t = oracle.build_table(s, 3.3)
    mu = oracle.random_dipoles(s.n, 9)
    a = oracle.tmatvec_thole(s, t, 3.0, 0.39, mu)
    b = oracle.tmatvec_ewald(s, t, 0.0, 3.0, 0.39, mu)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()
    a = oracle.perm_field_thole(s, t, 3.0, 0.39)
    b = oracle.perm_field_ewald(s, t, 0.0, 3.0, 0.39, exclude=False)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


def test_T_symmetric_ewald(oracle):
    """proj/tests/test_polar.cpp:267-296, for the Ewald + Thole T."""
    s = oracle.generate_system("uniform", 15, (9, 9, 9), 6)
    t = oracle.build_table(s, 3.0)
    n = 3 * s.n
    T = np.zeros((n, n))
    for c in range(n):
        mu = np.zeros((s.n, 3))
        mu[c // 3, c % 3] = 1.0
        T[:, c] = oracle.tmatvec_ewald(s, t, 0.6, 3.0, 0.39, mu).reshape(-1)
    assert np.abs(T - T.T).max() <= 1e-14


def mpole_system(oracle, n=12, box=40.0, seed=3, cluster=6.0):
    """A small cluster in a large box: no periodic image within the cutoff."""
    rng = np.random.default_rng(seed)
    pos = box / 2 + rng.uniform(-cluster / 2, cluster / 2, (n, 3))
    one = np.ones(n)
    s = System((box,) * 3, pos[:, 0].copy(), pos[:, 1].copy(), pos[:, 2].copy(),
               rng.uniform(-0.5, 0.5, n), one, one, one, one, rng.uniform(0.5, 1.5, n))
    s.dipole = rng.normal(0, 0.2, (n, 3))
    q = rng.normal(0, 0.1, (n, 6))
    tr = (q[:, 0] + q[:, 3] + q[:, 5]) / 3
    q[:, 0] -= tr
    q[:, 3] -= tr
    q[:, 5] -= tr
    s.quadrupole = q
    s.molecule = (np.arange(n) // 3).astype(np.int32)
    return s


def test_mpole_reduces_to_ewald_charges(oracle):
    """mu = Theta = 0: the multipole kernel equals the reference charge kernel."""
    s = oracle.generate_system("uniform", 200, (12, 12, 12), 2)
    t = oracle.build_table(s, 3.7)
    fo, eo, wo = oracle.ewald_real(s, t, 0.4, 3.7, 2.0)
    f, tq, e, w = oracle.mpole(s, t, 0.4, 3.7, 2.0, exclude=False)
    assert e == pytest.approx(eo, rel=1e-12)
    assert np.abs(f - fo).max() <= 1e-11 * np.abs(fo).max()
    assert np.abs(tq).max() == 0.0
    assert np.abs(w - wo).max() <= 1e-11 * np.abs(wo).max()


@pytest.mark.parametrize("alpha", [0.0, 0.45])
def test_mpole_forces_are_gradients(oracle, alpha):
    s = mpole_system(oracle)
    t = oracle.build_table(s, 9.0)
    f, tq, e, w = oracle.mpole(s, t, alpha, 9.0)
    num = fd_forces(lambda q: oracle.mpole(q, t, alpha, 9.0)[2], s, h=1e-6)
    assert np.abs(num - f).max() <= 1e-6 * max(1.0, np.abs(f).max())


def rotate_site(s, i, axis, ang):
    c, sn = np.cos(ang), np.sin(ang)
    k = np.zeros(3)
    k[axis] = 1.0
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    R = np.eye(3) + sn * K + (1 - c) * K @ K
    q = s.copy()
    q.dipole[i] = R @ s.dipole[i]
    Q6 = s.quadrupole[i]
    Q = np.array([[Q6[0], Q6[1], Q6[2]], [Q6[1], Q6[3], Q6[4]], [Q6[2], Q6[4], Q6[5]]])
    Qr = R @ Q @ R.T
    q.quadrupole[i] = [Qr[0, 0], Qr[0, 1], Qr[0, 2], Qr[1, 1], Qr[1, 2], Qr[2, 2]]
    return q


@pytest.mark.parametrize("alpha", [0.0, 0.45])
def test_mpole_torques_by_rotation(oracle, alpha):
    s = mpole_system(oracle, seed=5)
    t = oracle.build_table(s, 9.0)
    _, tq, _, _ = oracle.mpole(s, t, alpha, 9.0)
    h = 1e-6
    for i in (0, 4, 7):
        for a in range(3):
            up = oracle.mpole(rotate_site(s, i, a, h), t, alpha, 9.0)[2]
            dn = oracle.mpole(rotate_site(s, i, a, -h), t, alpha, 9.0)[2]
            assert tq[i, a] == pytest.approx(-(up - dn) / (2 * h), abs=1e-6 * max(1, np.abs(tq).max()))


def test_mpole_rotational_invariance(oracle):
    s = mpole_system(oracle, seed=8)
    t = oracle.build_table(s, 9.0)
    f, tq, e, _ = oracle.mpole(s, t, 0.3, 9.0)
    rng = np.random.default_rng(1)
    A = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    if np.linalg.det(A) < 0:
        A[:, 0] *= -1
    c = np.array(s.box) / 2
    q = s.copy()
    P = (np.stack([s.x, s.y, s.z], 1) - c) @ A.T + c
    q.x, q.y, q.z = P[:, 0].copy(), P[:, 1].copy(), P[:, 2].copy()
    q.dipole = s.dipole @ A.T
    for i in range(s.n):
        Q6 = s.quadrupole[i]
        Q = np.array([[Q6[0], Q6[1], Q6[2]], [Q6[1], Q6[3], Q6[4]], [Q6[2], Q6[4], Q6[5]]])
        Qr = A @ Q @ A.T
        q.quadrupole[i] = [Qr[0, 0], Qr[0, 1], Qr[0, 2], Qr[1, 1], Qr[1, 2], Qr[2, 2]]
    f2, tq2, e2, _ = oracle.mpole(q, oracle.build_table(q, 9.0), 0.3, 9.0)
    assert e2 == pytest.approx(e, rel=1e-12)
    assert np.abs(f2 - f @ A.T).max() <= 1e-11 * np.abs(f).max()
    assert np.abs(tq2 - tq @ A.T).max() <= 1e-11 * np.abs(tq).max()


def test_field_is_minus_dU_dmu(oracle):
    """dU/dmu_i = -E_i: ties the tensor field to the tensor energy; and the
    Thole/Ewald field code equals the tensor field when Thole is off."""
    s = mpole_system(oracle, seed=2)
    s.molecule = None
    t = oracle.build_table(s, 9.0)
    E = oracle.mpole_field_tensor(s, t, 0.4, 9.0, exclude=False)
    h = 1e-6
    for i in (1, 5):
        for a in range(3):
            up, dn = s.copy(), s.copy()
            up.dipole[i, a] += h
            dn.dipole[i, a] -= h
            d = (oracle.mpole(up, t, 0.4, 9.0, exclude=False)[2]
                 - oracle.mpole(dn, t, 0.4, 9.0, exclude=False)[2]) / (2 * h)
            assert d == pytest.approx(-E[i, a], abs=1e-7 * max(1, np.abs(E).max()))
    E2 = oracle.perm_field_ewald(s, t, 0.4, 9.0, 1e12, exclude=False)  # l3,l5,l7 -> 1
    assert np.abs(E2 - E).max() <= 1e-11 * np.abs(E).max()


def test_pcg_matches_dense_solve(oracle):
    """Method of proj/tests/test_polar.cpp:298-376 with the Ewald T and PCG."""
    for n in (6, 15):
        s = oracle.generate_system("uniform", n, (9, 9, 9), 21)
        t = oracle.build_table(s, 3.0)
        m = 3 * n
        A = np.zeros((m, m))
        for c in range(m):
            mu = np.zeros((n, 3))
            mu[c // 3, c % 3] = 1.0
            A[:, c] = -oracle.tmatvec_ewald(s, t, 0.5, 3.0, 0.39, mu).reshape(-1)
        A += np.diag(np.repeat(1.0 / s.polarizability, 3))
        E = oracle.perm_field_ewald(s, t, 0.5, 3.0, 0.39, exclude=False)
        x = np.linalg.solve(A, E.reshape(-1)).reshape(n, 3)
        mu, it, rms = oracle.pcg(s, t, 0.5, 3.0, 0.39, E, 1e-12, 200)
        assert np.abs(mu - x).max() <= 1e-9 * np.abs(x).max()


def test_pcg_zero_field_is_converged(oracle):
    """Edge case: no permanent field (no pairs, or all charges zero) --
    mu = 0 after one step, no 0/0 in a_k or beta."""
    s = oracle.generate_system("uniform", 15, (9, 9, 9), 21)
    t = oracle.build_table(s, 3.0)
    mu, it, rms = oracle.pcg(s, t, 0.5, 3.0, 0.39, np.zeros((15, 3)), 1e-5, 10)
    assert np.isfinite(mu).all() and not np.any(mu) and rms == 0.0 and it == 1


def test_pcg_agrees_with_jacobi_where_it_converges(oracle):
    s = oracle.generate_system("uniform", 15, (9, 9, 9), 21)
    t = oracle.build_table(s, 3.0)
    mj, _ = oracle.jacobi(s, t, 3.0, 0.39, 1e-12, 500)
    E = oracle.perm_field_thole(s, t, 3.0, 0.39)
    mp, _, _ = oracle.pcg(s, t, 0.0, 3.0, 0.39, E, 1e-12, 200)
    assert np.abs(mp - mj).max() <= 1e-9 * np.abs(mj).max()


def test_reduce_sites_and_chain_rule(oracle):
    """H-reduction: Halgren forces on atoms = -dE/dx of the reduced-site energy."""
    rng = np.random.default_rng(4)
    n = 12
    s = mpole_system(oracle, n=n, seed=4)
    s.hal_r0 = rng.uniform(2.5, 3.5, n)
    s.hal_epsilon = rng.uniform(0.01, 0.1, n)
    parent = np.array([3 * (i // 3) for i in range(n)], np.int32)
    factor = np.where(np.arange(n) % 3 == 0, 1.0, 0.91)

    def energy_forces(q):
        xr, yr, zr = oracle.reduce_sites(q, parent, factor)
        r = q.copy()
        r.x, r.y, r.z = xr, yr, zr
        fr, e, _ = oracle.halgren(r, oracle.build_table(r, 9.0), 9.0)
        return e, oracle.reduce_forces(parent, factor, fr)

    e, f = energy_forces(s)
    num = fd_forces(lambda q: energy_forces(q)[0], s)
    assert np.abs(num - f).max() <= 1e-6 * max(1.0, np.abs(f).max())


def test_fast_port_matches_tensor_oracle(oracle):
    """The closed-form CPU port (CPU-baseline leg) == the T-tensor oracle; this
    also checks, on CPU, the closed forms the CUDA kernels use."""
    from oracle.oracle import FastPort
    fp = FastPort()
    s = mpole_system(oracle, n=30, seed=11, cluster=9.0)
    t = oracle.build_table(s, 9.0)
    for alpha in (0.0, 0.5):
        fo, to, eo, wo = oracle.mpole(s, t, alpha, 8.0, 2.0, exclude=True)
        f, tq, e = fp.mpole(s, t, alpha, 8.0, 2.0, exclude=True)
        assert e == pytest.approx(eo, rel=1e-12)
        assert np.abs(fp.last_virial - wo).max() <= 1e-11 * np.abs(wo).max()
        assert np.abs(f - fo).max() <= 1e-11 * np.abs(fo).max()
        assert np.abs(tq - to).max() <= 1e-11 * np.abs(to).max()
        eo = oracle.perm_field_ewald(s, t, alpha, 8.0, 0.39, exclude=True)
        assert np.abs(fp.perm_field(s, t, alpha, 8.0, 0.39, True) - eo).max() <= 1e-12 * np.abs(eo).max()
        mu = s.dipole
        eo = oracle.tmatvec_ewald(s, t, alpha, 8.0, 0.39, mu)
        assert np.abs(fp.tmatvec(s, t, alpha, 8.0, 0.39, mu) - eo).max() <= 1e-12 * np.abs(eo).max()


# ---------------------------------------------------------------- polarization forces
def _epol(oracle, s, t, alpha, thole=0.39, cutoff=9.0, electric=1.0):
    """E_pol = -1/2 mu*.E_perm at the (tightly) converged dipoles."""
    ep = oracle.perm_field_ewald(s, t, alpha, cutoff, thole, exclude=True)
    mu, _, _ = oracle.pcg(s, t, alpha, cutoff, thole, ep, 1e-13, 1000)
    return -0.5 * electric * float(np.sum(mu * ep)), mu, ep


@pytest.mark.parametrize("alpha", [0.0, 0.45])
def test_polar_energy_is_variational(oracle, alpha):
    """At the solution, sum U_ij + 1/2 mu.alpha^-1.mu == -1/2 mu.E_perm."""
    s = mpole_system(oracle, seed=11)
    t = oracle.build_table(s, 9.0)
    e, mu, ep = _epol(oracle, s, t, alpha)
    _, _, epair, _ = oracle.polar_forces(s, t, alpha, 9.0, 0.39, mu)
    eself = 0.5 * float(np.sum(mu * mu / s.polarizability[:, None]))
    assert epair + eself == pytest.approx(e, rel=1e-9)


@pytest.mark.parametrize("alpha", [0.0, 0.45])
def test_polar_forces_are_gradients(oracle, alpha):
    """Forces at fixed mu == -dE_pol/dr with mu re-solved at every displacement
    (the Hellmann-Feynman property of the stationary polarization energy)."""
    s = mpole_system(oracle, seed=12)
    t = oracle.build_table(s, 9.0)
    _, mu, _ = _epol(oracle, s, t, alpha)
    f, _, _, w = oracle.polar_forces(s, t, alpha, 9.0, 0.39, mu)
    num = fd_forces(lambda q: _epol(oracle, q, t, alpha)[0], s, h=1e-5)
    assert np.abs(num - f).max() <= 2e-6 * max(1.0, np.abs(f).max())
    # momentum conservation (pair forces); the pair virial of these
    # non-central forces is not symmetric
    assert np.abs(f.sum(0)).max() <= 1e-10 * np.abs(f).max()


@pytest.mark.parametrize("alpha", [0.0, 0.45])
def test_polar_torques_by_rotation(oracle, alpha):
    """Torque on the permanent multipoles == -dE_pol/dtheta (re-solved)."""
    s = mpole_system(oracle, seed=13)
    t = oracle.build_table(s, 9.0)
    _, mu, _ = _epol(oracle, s, t, alpha)
    _, tq, _, _ = oracle.polar_forces(s, t, alpha, 9.0, 0.39, mu)
    h = 1e-5
    for i in (1, 5, 9):
        for a in range(3):
            up = _epol(oracle, rotate_site(s, i, a, h), t, alpha)[0]
            dn = _epol(oracle, rotate_site(s, i, a, -h), t, alpha)[0]
            assert tq[i, a] == pytest.approx(-(up - dn) / (2 * h),
                                             abs=2e-6 * max(1, np.abs(tq).max()))


# ---------------------------------------------------------------- local frames (8(f)#2)
def water_cluster(n_mol=4, seed=21, box=40.0, spread=6.0):
    """n_mol rigid waters (O-H 0.9572 A, 104.52 deg) scattered in a cluster
    in a large box, random local-frame multipoles, frames per water_frames."""
    from oracle import frames as fr
    rng = np.random.default_rng(seed)
    pos = []
    th = np.deg2rad(104.52) / 2
    for _ in range(n_mol):
        o = box / 2 + rng.uniform(-spread / 2, spread / 2, 3)
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        h1 = o + 0.9572 * q @ np.array([np.sin(th), 0, np.cos(th)])
        h2 = o + 0.9572 * q @ np.array([-np.sin(th), 0, np.cos(th)])
        pos += [o, h1, h2]
    pos = np.array(pos)
    n = len(pos)
    one = np.ones(n)
    charge = np.tile([-0.51966, 0.25983, 0.25983], n_mol)
    s = System((box,) * 3, pos[:, 0].copy(), pos[:, 1].copy(), pos[:, 2].copy(), charge, one,
               one, one, one, np.tile([0.837, 0.496, 0.496], n_mol))
    s.molecule = (np.arange(n) // 3).astype(np.int32)
    dl = rng.normal(0, 0.15, (n, 3))
    ql = rng.normal(0, 0.1, (n, 6))
    tr = (ql[:, 0] + ql[:, 3] + ql[:, 5]) / 3
    ql[:, 0] -= tr
    ql[:, 3] -= tr
    ql[:, 5] -= tr
    frame, za, xa = fr.water_frames(s.molecule)
    return s, frame, za, xa, dl, ql


def _framed(s, frame, za, xa, dl, ql):
    from oracle import frames as fr
    q = s.copy()
    pos = np.stack([q.x, q.y, q.z], 1)
    q.dipole, q.quadrupole = fr.rotate(pos, q.box, frame, za, xa, dl, ql)
    return q


@pytest.mark.parametrize("alpha", [0.0, 0.45])
def test_frame_forces_are_gradients(oracle, alpha):
    """With local frames the total force -- translational multipole force plus
    the frame atoms' share of the torques -- is -dE/dr with the frames
    rebuilt at every displacement."""
    from oracle import frames as fr
    s, frame, za, xa, dl, ql = water_cluster()
    t = oracle.build_table(s, 9.0)
    g = _framed(s, frame, za, xa, dl, ql)
    f, tq, e, _ = oracle.mpole(g, t, alpha, 9.0)
    pos = np.stack([s.x, s.y, s.z], 1)
    ftot = f + fr.torque_forces(pos, s.box, frame, za, xa, tq)
    num = fd_forces(lambda q: oracle.mpole(_framed(q, frame, za, xa, dl, ql), t, alpha, 9.0)[2],
                    s, h=1e-6)
    assert np.abs(num - ftot).max() <= 1e-6 * max(1.0, np.abs(ftot).max())
    assert np.abs(ftot.sum(0)).max() <= 1e-10 * np.abs(ftot).max()


# ---------------------------------------------------------------- reciprocal space (8(f)#3)
def test_ewald_oracle_is_alpha_independent(oracle):
    """Real space (oracle mdo_ewald_real) + direct reciprocal sum + self +
    excluded-pair terms: the full Ewald energy and forces do not depend on
    the splitting parameter (the oracle/ewald_recip.py pin)."""
    from oracle import ewald_recip as er
    n_mol, L = 30, 20.0
    s = oracle.generate_system("uniform", 3 * n_mol, (L, L, L), 3, 1.0)
    s.charge[:] = np.tile([-0.8, 0.4, 0.4], n_mol)
    s.molecule = (np.arange(3 * n_mol) // 3).astype(np.int32)
    pos = np.stack([s.x, s.y, s.z], 1)
    t = oracle.build_table(s, 9.9)
    tot = []
    for a in (0.5, 0.6):
        fr_, er_, _ = oracle.ewald_real(s, t, a, 9.9, 1.0, exclude=True)
        e2, f2, _ = er.recip(pos, s.charge, s.box, a, kmax=(24, 24, 24))
        e4, f4, _ = er.excluded_correction(pos, s.charge, s.box, s.molecule, a)
        tot.append((er_ + e2 + er.self_energy(s.charge, a) + e4, fr_ + f2 + f4))
    assert abs(tot[0][0] - tot[1][0]) <= 1e-11
    assert np.abs(tot[0][1] - tot[1][1]).max() <= 1e-10
    # forces are -dE/dr (finite differences of the reciprocal sum)
    e0, f0, _ = er.recip(pos, s.charge, s.box, 0.5, kmax=(16, 16, 16))
    h = 1e-6
    for i, a in ((0, 0), (7, 1), (40, 2)):
        p1, p2 = pos.copy(), pos.copy()
        p1[i, a] += h
        p2[i, a] -= h
        num = -(er.recip(p1, s.charge, s.box, 0.5, (16, 16, 16))[0] -
                er.recip(p2, s.charge, s.box, 0.5, (16, 16, 16))[0]) / (2 * h)
        assert num == pytest.approx(f0[i, a], abs=1e-7)


# ---------------------------------------------------------------- MD loop (8(f)#4)
def test_bonded_oracle_forces_are_gradients(oracle):
    from oracle import md
    s, *_ = water_cluster(n_mol=3, seed=5)
    pos = np.stack([s.x, s.y, s.z], 1) + np.random.default_rng(2).normal(0, 0.05, (9, 3))
    b, a = md.water_topology(3)
    args = (b, 529.6, 0.9572, a, 34.05, np.deg2rad(104.52))
    _, _, f = md.bonded(pos, s.box, *args)
    h = 1e-6
    for i in range(9):
        for k in range(3):
            p1, p2 = pos.copy(), pos.copy()
            p1[i, k] += h
            p2[i, k] -= h
            e1 = sum(md.bonded(p1, s.box, *args)[:2])
            e2 = sum(md.bonded(p2, s.box, *args)[:2])
            assert -(e1 - e2) / (2 * h) == pytest.approx(f[i, k], abs=1e-6)


# ------------------------------------------------------- water fixture twin
@pytest.mark.parametrize("model,n_mol,box,seed", [("amoeba", 1000, 31.04, 3),
                                                  ("charmm", 1000, 31.04, 1),
                                                  ("amoeba", 333, 21.5, 7)])
def test_water_fixture_twin_is_bit_identical(oracle, mdg, model, n_mol, box, seed):
    """The oracle's generator (mdo_water_generate) reproduces the product's
    mdg_water_generate bit for bit, so the CPU reference arm builds the same
    fixture without loading the product library."""
    s, par, fac = oracle.water_box(n_mol, box, seed, model)
    p = mdg.water_box(n_mol, box, seed, model)
    for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
              "polarizability", "molecule"):
        assert np.array_equal(getattr(s, k), getattr(p, k)), k
    if model == "amoeba":
        assert np.array_equal(s.dipole, p.dipole) and np.array_equal(s.quadrupole, p.quadrupole)
        assert np.array_equal(par, p.hred_parent) and np.array_equal(fac, p.hred_factor)
        for a, b in zip(oracle.reduce_sites(s, par, fac), mdg.reduce_sites_host(p)):
            assert np.array_equal(a, b)


def test_rows_for_sites_match_brute_force(oracle):
    """The sampled-row oracle of the config-4 parity test (cell candidates +
    the reference predicate) == the O(N^2) brute-force pair set."""
    for n_mol, box, cut in ((1000, 31.04, 9.0), (300, 20.0, 9.0), (2000, 39.1, 11.0)):
        s, _, _ = oracle.water_box(n_mol, box, 1, "amoeba")
        sites = np.arange(0, 3 * n_mol, 7)
        bf = oracle.brute_force_pairs(s, cut)
        for i, r in zip(sites, oracle.rows_for_sites(s, cut, sites)):
            want = np.sort(np.concatenate([bf[bf[:, 0] == i, 1], bf[bf[:, 1] == i, 0]]))
            np.testing.assert_array_equal(r, want)


# ------------------------------------------------ multipole Ewald oracle (8(f)#3)
def _mp_water(oracle):
    s, _, _ = oracle.water_box(27, 10.2, 3, "amoeba")
    return s


def test_mpole_ewald_oracle_forces_torques_by_fd(oracle):
    """oracle/ewald_mpole.py: reciprocal + self + excluded forces == -dE/dr and
    torques == -dE/dtheta (finite differences / rotations of one site)."""
    from oracle import ewald_mpole as em
    s = _mp_water(oracle)
    pos = np.stack([s.x, s.y, s.z], 1)

    def energy(p, mu=s.dipole, q6=s.quadrupole):
        e = em.recip(p, s.charge, mu, q6, s.box, 0.6, kmax=(8, 8, 8), energy_only=True)[0]
        return e + em.excluded_correction(p, s.charge, mu, q6, s.box, s.molecule, 0.6,
                                          pair=em.mpole_pair)[0]

    _, f, t = em.recip(pos, s.charge, s.dipole, s.quadrupole, s.box, 0.6, kmax=(8, 8, 8))
    _, fx, tx = em.excluded_correction(pos, s.charge, s.dipole, s.quadrupole, s.box,
                                       s.molecule, 0.6, pair=em.mpole_pair)
    f, t = f + fx, t + tx
    h = 1e-5
    for i, k in ((0, 0), (4, 1), (13, 2)):
        p = pos.copy()
        p[i, k] += h
        ep = energy(p)
        p[i, k] -= 2 * h
        assert f[i, k] == pytest.approx(-(ep - energy(p)) / (2 * h), rel=1e-6, abs=1e-9)

    def rot(ax, th):
        ax = np.asarray(ax, float) / np.linalg.norm(ax)
        K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
        return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K

    for i, ax in ((2, (0, 0, 1)), (7, (1, 1, 0))):
        vals = []
        for th in (h, -h):
            R = rot(ax, th)
            m2 = s.dipole.copy()
            m2[i] = R @ s.dipole[i]
            Q = R @ em.quad3(s.quadrupole)[i] @ R.T
            q6 = s.quadrupole.copy()
            q6[i] = [Q[0, 0], Q[0, 1], Q[0, 2], Q[1, 1], Q[1, 2], Q[2, 2]]
            vals.append(energy(pos, m2, q6))
        ax = np.asarray(ax, float) / np.linalg.norm(ax)
        assert t[i] @ ax == pytest.approx(-(vals[0] - vals[1]) / (2 * h), rel=1e-5, abs=1e-9)


def test_mpole_ewald_total_is_alpha_independent(oracle):
    """Real space (mdo.c tensor multipoles, exclusions) + reciprocal + self +
    excluded pairs: one energy for two splitting parameters (both sums
    converged: erfc(a rc) < 1e-9, k-space tail < 1e-12)."""
    from oracle import ewald_mpole as em
    s = _mp_water(oracle)
    pos = np.stack([s.x, s.y, s.z], 1)
    t = oracle.build_table(s, 4.9)
    tot = []
    for a in (0.95, 1.05):
        er = oracle.mpole(s, t, a, 4.9, 1.0, exclude=True)[2]
        ek = em.recip(pos, s.charge, s.dipole, s.quadrupole, s.box, a, kmax=(17, 17, 17),
                      energy_only=True)[0]
        es = em.self_energy(s.charge, s.dipole, s.quadrupole, a)
        ex = em.excluded_correction(pos, s.charge, s.dipole, s.quadrupole, s.box, s.molecule,
                                    a, pair=em.mpole_pair)[0]
        tot.append(er + ek + es + ex)
    assert tot[0] == pytest.approx(tot[1], rel=2e-7)
