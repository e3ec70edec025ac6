"""BAOAB-RESPA (mdg.h mdg_md_run, MDG_INTEGRATOR_BAOAB_RESPA): the two-level
multi-timestep Langevin integrator of the paper's Rel2
(bonded terms in the inner level,
nonbonded in the outer). CPU: the oracle's counter-based noise. GPU: the
device trajectory against oracle/md.py baoab_respa driven by the oracle's
forces, NVE energy conservation with friction 0, and the thermostat's
temperature; and energy conservation of the whole AMOEBA force chain
(frames, torques, polarization forces) under both integrators."""
import numpy as np
import pytest

from conftest import to_oracle_system

BOND_ARGS = (529.6, 0.9572, 34.05, np.deg2rad(104.52))


def test_oracle_noise_is_standard_normal_and_counter_based():
    from oracle import md
    g = md.gauss(7, 0, 200_000)
    assert g.shape == (200_000, 3)
    assert abs(g.mean()) < 0.01 and abs(g.std() - 1.0) < 0.01
    # fourth moment of a normal is 3
    assert abs((g ** 4).mean() - 3.0) < 0.05
    np.testing.assert_array_equal(md.gauss(7, 0, 50), g[:50])  # per-site streams
    assert not np.array_equal(md.gauss(7, 1, 50), g[:50])      # counter
    assert not np.array_equal(md.gauss(8, 0, 50), g[:50])      # seed


def test_oracle_respa_one_inner_step_nve_is_velocity_verlet():
    """With one inner step, friction 0 and no fast forces the scheme is
    velocity Verlet (the A(h/2) A(h/2) split aside)."""
    from oracle import md
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 10, (20, 3))
    vel = rng.normal(0, 0.01, (20, 3))
    mass = np.full(20, 12.0)
    k = 0.5

    def slow(p):  # harmonic well around the box centre
        d = p - 5.0
        return -2 * k * d, float(k * (d * d).sum())

    def fast(p):
        return np.zeros_like(p), 0.0

    p1, v1, ek1, ep1 = md.baoab_respa(pos, vel, mass, (10, 10, 10), slow, fast, 0.5, 1, 0.0,
                                      300.0, 1, 30)
    p2, v2, ek2, ep2 = md.velocity_verlet(pos, vel, mass, (10, 10, 10), slow, 0.5, 30)
    np.testing.assert_allclose(p1, p2, atol=1e-12)
    np.testing.assert_allclose(v1, v2, atol=1e-14)
    np.testing.assert_allclose(ep1, ep2, rtol=1e-10)


def _setup(engine, mdg, n_mol=216, box=18.6, seed=2, temp=300.0):
    from test_gpu_parity import _md_water
    s, mass, vel, b, a = _md_water(mdg, n_mol, box, seed, temp)
    engine.upload_system(s)
    engine.upload_bonded(b, BOND_ARGS[0], BOND_ARGS[1], a, BOND_ARGS[2], BOND_ARGS[3])
    engine.upload_velocities(vel, mass)
    return s, mass, vel, b, a


def _respa(mdg, nsteps, dt, inner, friction, temp, seed, rebuild_every=10):
    p = mdg.MDParams(0, nsteps, dt, rebuild_every, 0, 1, 9.3, 0.0, 1)
    p.integrator = mdg.INTEGRATOR_BAOAB_RESPA
    p.inner_steps = inner
    p.friction_ps = friction
    p.temperature_k = temp
    p.seed = seed
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("friction,resort", [(0.0, "20"), (5.0, "1")])
def test_respa_trajectory_matches_oracle(engine, oracle, mdg, friction, resort, monkeypatch):
    """12 outer steps of 1 fs (4 bonded sub-steps of 0.25 fs), with and
    without the Langevin O step, against the numpy integrator on the oracle's
    forces and the same noise stream: positions within 1e-9 A. The Langevin
    case re-sorts the sites at each list rebuild (MDG_RESORT=1): the noise
    follows the caller's site ids, not the device order."""
    from oracle import md
    monkeypatch.setenv("MDG_RESORT", resort)
    s, mass, vel, b, a = _setup(engine, mdg)
    so = to_oracle_system(s)
    bond_args = (b, BOND_ARGS[0], BOND_ARGS[1], a, BOND_ARGS[2], BOND_ARGS[3])

    def slow(pos):
        q = so.copy()
        q.x[:], q.y[:], q.z[:] = pos[:, 0], pos[:, 1], pos[:, 2]
        t = oracle.build_table(q, 9.3)
        f1, e1, _ = oracle.lj(q, t, 8.0, shift=True, exclude=True)
        f2, e2, _ = oracle.ewald_real(q, t, 0.45, 8.0, mdg.ELECTRIC, exclude=True)
        return f1 + f2, e1 + e2

    def fast(pos):
        eb, ea, f = md.bonded(pos, so.box, *bond_args)
        return f, eb + ea

    pos0 = np.stack([s.x, s.y, s.z], 1)
    p_o, v_o, ek_o, ep_o = md.baoab_respa(pos0, vel, mass, so.box, slow, fast, 1.0, 4, friction,
                                          300.0, 11, 12)
    p = _respa(mdg, 12, 1.0, 4, friction, 300.0, 11)
    ek, ep = engine.md_run(p, charmm=mdg.CharmmParams(8.0, 0.45, mdg.ELECTRIC, 1, 1))
    pos = engine.fetch_positions()
    d = pos - p_o
    d -= np.asarray(so.box) * np.rint(d / np.asarray(so.box))
    assert np.abs(d).max() <= 1e-9
    assert np.abs(engine.fetch_velocities() - v_o).max() <= 1e-9 * np.abs(v_o).max()
    np.testing.assert_allclose(ek, ek_o, rtol=1e-9)
    np.testing.assert_allclose(ep, ep_o, rtol=1e-9)


@pytest.mark.gpu
def test_respa_nve_conserves_energy_at_a_longer_outer_step(engine, mdg):
    """Friction 0, 1 fs outer step with the O-H vibrations in 4 sub-steps:
    over 1,000 fs the total energy stays within 3e-3 of the kinetic energy
    (the unrelaxed fixture heats from 300 K to ~750 K meanwhile), and over
    the first 250 fs its spread is under 0.3x that of velocity Verlet at the
    same 1 fs step (measured: 2.74 vs 18.1 kcal/mol; velocity Verlet at
    0.25 fs: 1.07)."""
    ch = mdg.CharmmParams(8.0, 0.45, mdg.ELECTRIC, 1, 1)
    _setup(engine, mdg, seed=4)
    ek, ep = engine.md_run(_respa(mdg, 1000, 1.0, 4, 0.0, 0.0, 0, 5), charmm=ch)
    et = ek + ep
    assert np.all(np.isfinite(et))
    assert (et.max() - et.min()) <= 3e-3 * ek.mean(), (et.max() - et.min(), ek.mean())
    spread_respa = et[:250].max() - et[:250].min()
    _setup(engine, mdg, seed=4)
    ek, ep = engine.md_run(mdg.MDParams(0, 250, 1.0, 5, 0, 1, 9.3, 0.0, 1), charmm=ch)
    et = ek + ep
    assert spread_respa <= 0.3 * (et.max() - et.min()), (spread_respa, et.max() - et.min())


@pytest.mark.gpu
def test_respa_langevin_holds_the_bath_temperature(engine, mdg):
    """Friction 20/ps at 350 K from a 300 K start: the kinetic temperature
    averaged over the last 2,000 of 3,000 outer steps is 350 K within 4 %."""
    s, mass, vel, b, a = _setup(engine, mdg, seed=5)
    ek, ep = engine.md_run(_respa(mdg, 3000, 1.0, 4, 20.0, 350.0, 99, 20),
                           charmm=mdg.CharmmParams(8.0, 0.45, mdg.ELECTRIC, 1, 1))
    n = s.n_sites
    t_inst = 2.0 * ek / (3 * n * 0.0019872041)
    assert np.all(np.isfinite(t_inst))
    assert abs(t_inst[1000:].mean() - 350.0) <= 0.04 * 350.0, t_inst[1000:].mean()


@pytest.mark.gpu
def test_respa_bad_parameters_are_contract_violations(engine, mdg):
    _setup(engine, mdg, 27, 9.4, 3)
    ch = mdg.CharmmParams(4.0, 0.45, mdg.ELECTRIC, 1, 1)

    def params(inner, friction, integrator=None):
        p = _respa(mdg, 2, 1.0, inner, friction, 300.0, 1, 1)
        p.elec_list_cutoff = 4.6
        if integrator is not None:
            p.integrator = integrator
        return p

    engine.md_run(params(2, 1.0), charmm=ch)  # the valid case runs
    for bad in (params(0, 1.0), params(2, -1.0), params(2, 1.0, integrator=7)):
        with pytest.raises(mdg.ContractViolation):
            engine.md_run(bad, charmm=ch)


def _amoeba_water(engine, mdg, scale=0.1, n_mol=512, box=24.8):
    """The AMOEBA water fixture with its random multipoles at `scale` in
    local water frames (z-then-x on H, bisector on O), bonds/angles and
    300 K velocities. At full scale the random multipoles collapse H...O
    pairs within ~25 fs (the static benchmark's values are not a force
    field); at 1/10 the dynamics is stable."""
    s = mdg.water_box(n_mol, box, 2, "amoeba")
    n = s.n_sites
    frame = np.zeros(n, np.int32)
    za = np.zeros(n, np.int32)
    xa = np.zeros(n, np.int32)
    o = np.arange(0, n, 3)
    frame[o], za[o], xa[o] = 2, o + 1, o + 2
    frame[o + 1], za[o + 1], xa[o + 1] = 1, o, o + 2
    frame[o + 2], za[o + 2], xa[o + 2] = 1, o, o + 1
    mass = np.tile([15.999, 1.008, 1.008], n_mol)
    b = np.stack([np.repeat(o, 2), (o[:, None] + np.array([1, 2])).ravel()], 1)
    a = np.stack([o + 1, o, o + 2], 1)
    rng = np.random.default_rng(3)
    vel = rng.normal(size=(n, 3)) * np.sqrt(0.0019872041 * 300.0 * 4.184e-4 / mass)[:, None]
    engine.upload_system(s)
    engine.upload_frames(frame, za, xa, scale * np.asarray(s.dipole),
                         scale * np.asarray(s.quadrupole))
    engine.upload_bonded(b, BOND_ARGS[0], BOND_ARGS[1], a, BOND_ARGS[2], BOND_ARGS[3])
    engine.upload_velocities(vel, mass)
    return s



def _amoeba_params(mdg):
    t = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
    return mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-6, 100, 1, t)


@pytest.mark.gpu
def test_amoeba_nve_conserves_energy(engine, mdg):
    """The whole AMOEBA force chain in dynamics -- Halgren with H reduction,
    multipoles in rotating local frames (torques -> forces), the PCG-solved
    induced dipoles and their forces, bonds/angles -- conserves energy:
    2,000 velocity-Verlet steps of 0.25 fs, total energy within 3e-3 of the
    kinetic energy (measured 1.7e-3; the CHARMM test's bound is 2e-3), the
    first and last 200 steps within 1e-3 on average (measured 5.9e-4, the
    PCG's 1e-6 D tolerance)."""
    _amoeba_water(engine, mdg)
    try:
        ek, ep = engine.md_run(mdg.MDParams(1, 2000, 0.25, 20, 0, 1, 9.0, 11.0, 1),
                               amoeba=_amoeba_params(mdg))
    finally:
        engine.upload_frames(None, None, None)
    et = ek + ep
    assert np.all(np.isfinite(et))
    assert (et.max() - et.min()) <= 3e-3 * ek.mean(), (et.max() - et.min(), ek.mean())
    # no drift: the first and last 200 steps agree on average
    assert abs(et[-200:].mean() - et[:200].mean()) <= 1e-3 * ek.mean()


@pytest.mark.gpu
def test_amoeba_respa_nve_conserves_energy(engine, mdg):
    """BAOAB-RESPA with friction 0 on the same AMOEBA system: 500 outer
    steps of 1 fs (bonded terms in 4 sub-steps) keep the total energy within
    3e-3 of the kinetic energy."""
    _amoeba_water(engine, mdg)
    p = mdg.MDParams(1, 500, 1.0, 5, 0, 1, 9.0, 11.0, 1)
    p.integrator = mdg.INTEGRATOR_BAOAB_RESPA
    p.inner_steps = 4
    try:
        ek, ep = engine.md_run(p, amoeba=_amoeba_params(mdg))
    finally:
        engine.upload_frames(None, None, None)
    et = ek + ep
    assert np.all(np.isfinite(et))
    assert (et.max() - et.min()) <= 3e-3 * ek.mean(), (et.max() - et.min(), ek.mean())


@pytest.mark.gpu
def test_aspc_predictor_same_dynamics_fewer_iterations(engine, mdg, monkeypatch):
    """ASPC (mdg_md_params.predictor): the PCG of each MD step starts from
    dipoles extrapolated from the last six converged ones. The solve still
    runs to its tolerance, so the trajectory is the one without the
    predictor to within that tolerance, in fewer iterations. The sites are
    re-sorted at every list rebuild (the stored dipoles follow them)."""
    monkeypatch.setenv("MDG_RESORT", "1")
    out = {}
    for pred in (mdg.PREDICT_NONE, mdg.PREDICT_ASPC):
        _amoeba_water(engine, mdg)
        p = mdg.MDParams(1, 40, 0.25, 10, 0, 1, 9.0, 11.0, 1)
        p.predictor = pred
        try:
            ek, ep = engine.md_run(p, amoeba=_amoeba_params(mdg))
            e, w, it, rms = engine.fetch_energies()
            out[pred] = (engine.fetch_positions(), ek + ep, it)
        finally:
            engine.upload_frames(None, None, None)
    (x0, e0, it0), (x1, e1, it1) = out[mdg.PREDICT_NONE], out[mdg.PREDICT_ASPC]
    d = x1 - x0
    d -= 24.8 * np.rint(d / 24.8)
    assert np.abs(d).max() <= 1e-6
    np.testing.assert_allclose(e1, e0, rtol=1e-7)
    assert it1 < it0, (it1, it0)


@pytest.mark.gpu
def test_md_rebuilds_lists_early_when_sites_move_fast(engine, mdg):
    """A rebuild interval too long for the motion (1 fs steps, rebuild_every
    200, a 9.3 A list over an 8 A cutoff): mdg_md_run rebuilds early when the
    device flags a site past 0.6 x the list's tolerable motion, the run
    completes without an outdated-list error, and it matches the run with a
    short schedule to the dynamics' chaos over 100 fs."""
    out = {}
    for every in (200, 5):
        _setup(engine, mdg, seed=6)
        r0 = engine.md_rebuild_count()
        ek, ep = engine.md_run(mdg.MDParams(0, 100, 1.0, every, 0, 1, 9.3, 0.0, 1),
                               charmm=mdg.CharmmParams(8.0, 0.45, mdg.ELECTRIC, 1, 1))
        out[every] = (engine.md_rebuild_count() - r0, ek + ep)
    n_auto, e_auto = out[200]
    n_fixed, e_fixed = out[5]
    assert 1 < n_auto < n_fixed, (n_auto, n_fixed)
    np.testing.assert_allclose(e_auto[:20], e_fixed[:20], rtol=1e-6)
