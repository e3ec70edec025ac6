"""GPU: the multi-domain product path -- the C++ group runtime
(csrc/group.cu: halo refresh and summed CG scalars on the device inside the
PCG solve, csrc/polar.cu run_pcg_multi) over owned + halo domain contexts --
with 2, 4 and 8 domains hosted on ONE GPU (LOCAL backend: one process, one
shared stream, no kernel waits on another domain's), against the
single-domain engine; and the NCCL backend at world size 1."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HALO = 12.5  # 11 A vdW list + intramolecular extent + margin


def run_domains(mdg, s, size, params, lists, frames=None, steps=1, overlap=None, launches=None,
                recip=None):
    from paper_1906_01211_b200 import dd
    g = dd.DomainGroup(s, size, HALO, device=0, backend="local", list_cutoff=11.0,
                       overlap=overlap)
    try:
        assert g.check_halo(s)
        if frames is not None:
            g.upload_frames(*frames)
        if recip is not None:
            g.set_ewald_recip(*recip)
        tables = g.build_lists(lists)
        for _ in range(steps):
            g.amoeba_step(tables, params)
        en, w, it, rms = g.energies()
        ids, f = g.owned_forces()
        _, mu = g.owned_dipoles()
        if launches is not None:
            launches.append(g.launch_count())
    finally:
        g.close()
    n = s.n_sites
    F = np.zeros((n, 3))
    MU = np.zeros((n, 3))
    F[ids] = f
    MU[ids] = mu
    return F, MU, en, w, it


def single(mdg, s, p, frames=None, recip=None):
    with mdg.Engine(s.n_sites) as e:
        e.upload_system(s)
        if frames is not None:
            e.upload_frames(*frames)
        if recip is not None:
            e.set_ewald_recip(*recip)
        te = e.build_neighbor_table(9.0, list_id=0)
        tv = e.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
        e.amoeba_step(tv, te, p)
        en0, w0, it0, _ = e.fetch_energies()
        return en0, w0, it0, e.fetch_forces(), e.fetch_dipoles()



@pytest.mark.parametrize("size,polar_forces", [(2, False), (4, False), (8, False), (2, True)])
def test_domains_match_single_gpu(mdg, size, polar_forces):
    s = mdg.water_box(1728, 37.26, 5, "amoeba")
    terms = (mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
             if polar_forces else 0)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    en0, w0, it0, f0, mu0 = single(mdg, s, p)
    F, MU, en, w, it = run_domains(mdg, s, size, p, lists, steps=2)
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert np.allclose(w, w0, rtol=1e-9, atol=1e-9 * np.abs(w0).max())
    assert abs(it - it0) <= 1
    d = np.sqrt(np.mean(np.sum((MU - mu0) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-5


@pytest.mark.parametrize("size", [2, 8])
def test_interior_halo_overlap_matches(mdg, size):
    """Interior/halo overlap (mdg_group_set_overlap: each PCG iteration's
    halo refresh on the communication stream while the rows without halo
    sites run, then the boundary rows) gives the results of the serial
    exchange and of the single engine; the split adds the boundary
    mat-vec launches (and the per-step split)."""
    s = mdg.water_box(1728, 37.26, 7, "amoeba")
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    en0, w0, it0, f0, mu0 = single(mdg, s, p)
    runs, launches = {}, []
    for ov in (False, True):
        runs[ov] = run_domains(mdg, s, size, p, lists, steps=2, overlap=ov, launches=launches)
    F0, MU0, e0, _, i0 = runs[False]
    F1, MU1, e1, w1, i1 = runs[True]
    assert i1 == i0
    assert launches[1] > launches[0]
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F1 - F0).max() <= 1e-10 * rms
    assert np.abs(MU1 - MU0).max() <= 1e-10 * np.abs(MU0).max()
    assert np.abs(F1 - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert e1[k] == pytest.approx(en0[k], rel=1e-9)
    assert abs(i1 - it0) <= 1


@pytest.mark.parametrize("size,polar_forces", [(2, True), (4, False), (8, True)])
def test_domains_with_reciprocal_space(mdg, size, polar_forces):
    """Full Ewald in the decomposed step (replicated grid: owned sites spread
    per domain, grids summed, one transform, owned sites gathered): the
    multipole PME, the reciprocal field in the PCG operator and right-hand
    side and (with polarization forces) the combined permanent + induced
    pass match the single engine with the same grid."""
    s = mdg.water_box(1728, 37.26, 8, "amoeba")
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR
    if polar_forces:
        terms |= mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-6, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    recip = ((40, 40, 40), 5)
    en0, w0, it0, f0, mu0 = single(mdg, s, p, recip=recip)
    F, MU, en, w, it = run_domains(mdg, s, size, p, lists, steps=2, recip=recip)
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert abs(it - it0) <= 1
    d = np.sqrt(np.mean(np.sum((MU - mu0) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-6


@pytest.mark.parametrize("size,polar_forces", [(2, True), (3, False), (8, True)])
def test_domains_slab_fft(mdg, monkeypatch, size, polar_forces):
    """Slab-decomposed reciprocal space (MDG_PME_SLAB=1): grids reduced onto
    x-slabs, 2D transforms per slab, transpose to ky columns, 1D transforms
    along x and the convolution per part, and back; the parts' energy shares
    summed. Uneven slabs (42 x 36 x 30 over 3 and 8 parts) == the single
    engine's 3D transform at the same grid."""
    monkeypatch.setenv("MDG_PME_SLAB", "1")
    s = mdg.water_box(1728, 37.26, 8, "amoeba")
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR
    if polar_forces:
        terms |= mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-6, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    recip = ((42, 36, 30), 5)
    en0, w0, it0, f0, mu0 = single(mdg, s, p, recip=recip)
    F, MU, en, w, it = run_domains(mdg, s, size, p, lists, steps=2, recip=recip)
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert abs(it - it0) <= 1
    d = np.sqrt(np.mean(np.sum((MU - mu0) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-6


def test_nccl_group_slab_fft_world_size_one(mdg, monkeypatch):
    """The NCCL slab path (grouped ncclReduce, ncclSend/ncclRecv transposes,
    ncclBroadcast) at world size 1 with full Ewald == the single engine."""
    import os

    import torch.distributed as dist

    from paper_1906_01211_b200 import dd
    monkeypatch.setenv("MDG_PME_SLAB", "1")
    s = mdg.water_box(1000, 31.04, 8, "amoeba")
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-6, 100, 1, terms)
    recip = ((36, 36, 36), 5)
    en0, w0, it0, f0, mu0 = single(mdg, s, p, recip=recip)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29613"
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        g = dd.DomainGroup(s, 1, HALO, backend="nccl", rank=0, list_cutoff=11.0)
        try:
            g.set_ewald_recip(*recip)
            tables = g.build_lists([(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)])
            g.amoeba_step(tables, p)
            en, w, it, rms = g.energies()
            ids, f = g.owned_forces()
        finally:
            g.close()
    finally:
        dist.destroy_process_group()
    F = np.zeros_like(f0)
    F[ids] = f
    assert np.abs(F - f0).max() <= 1e-8 * np.sqrt(np.mean(f0 ** 2))
    assert abs(it - it0) <= 1
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)


def test_domains_with_local_frames(mdg):
    """Local multipole frames in the decomposed step (frame atoms mapped to
    each domain's local ids) match the single engine."""
    from oracle import frames as fr
    s = mdg.water_box(1728, 37.26, 6, "amoeba")
    frame, za, xa = fr.water_frames(s.molecule)
    frames = (frame, za, xa, np.asarray(s.dipole), np.asarray(s.quadrupole))
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    en0, w0, it0, f0, _ = single(mdg, s, p, frames)
    F, MU, en, w, it = run_domains(mdg, s, 2, p, lists, frames)
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert abs(it - it0) <= 1


def test_domains_follow_new_positions(mdg):
    """Positions moved within the halo margin: owned coordinates uploaded per
    domain, halos refreshed by the group exchange; == the single engine at
    the new coordinates."""
    from paper_1906_01211_b200 import dd
    s = mdg.water_box(1728, 37.26, 7, "amoeba")
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, 0)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    rng = np.random.default_rng(3)
    g = dd.DomainGroup(s, 2, HALO, backend="local", list_cutoff=11.0)
    try:
        tables = g.build_lists(lists)
        g.amoeba_step(tables, p)
        L = s.box[0]
        # within the halo margin ((12.5 - 11 - 1) / 2 = 0.25 A)
        x = np.mod(np.asarray(s.x) + rng.uniform(-0.12, 0.12, s.n_sites), L)
        y = np.mod(np.asarray(s.y) + rng.uniform(-0.12, 0.12, s.n_sites), L)
        z = np.mod(np.asarray(s.z) + rng.uniform(-0.12, 0.12, s.n_sites), L)
        g.update_positions(x, y, z)
        tables = g.build_lists(lists)
        g.amoeba_step(tables, p)
        en, _, it, _ = g.energies()
        ids, f = g.owned_forces()
        # past the margin: refused
        with pytest.raises(dd.HaloStale):
            g.update_positions(np.mod(x + 0.3, L), y, z)
    finally:
        g.close()
    s2 = mdg.water_box(1728, 37.26, 7, "amoeba")
    s2.x, s2.y, s2.z = x, y, z
    en0, _, it0, f0, _ = single(mdg, s2, p)
    F = np.zeros_like(f0)
    F[ids] = f
    assert np.abs(F - f0).max() <= 1e-8 * np.sqrt(np.mean(f0 ** 2))
    assert en[0] == pytest.approx(en0[0], rel=1e-9) and abs(it - it0) <= 1


def test_nccl_group_world_size_one(mdg):
    """The NCCL backend (ncclCommInitRank, in-place ncclAllReduce of the CG
    scalars, batched speculative iterations) at world size 1 on this GPU ==
    the single engine."""
    import os

    import torch.distributed as dist

    from paper_1906_01211_b200 import dd
    s = mdg.water_box(1000, 31.04, 8, "amoeba")
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, 0)
    en0, w0, it0, f0, mu0 = single(mdg, s, p)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29611")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        g = dd.DomainGroup(s, 1, HALO, backend="nccl", rank=0, list_cutoff=11.0)
        try:
            tables = g.build_lists([(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)])
            g.amoeba_step(tables, p)
            en, w, it, rms = g.energies()
            ids, f = g.owned_forces()
        finally:
            g.close()
    finally:
        dist.destroy_process_group()
    F = np.zeros_like(f0)
    F[ids] = f
    assert np.abs(F - f0).max() <= 1e-12 * np.abs(f0).max()
    assert it == it0 and rms < 1e-5
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-12)


def test_domains_replan_after_migration(mdg):
    """Molecules moved past the halo margin (whole molecules shifted by 3 A,
    so many change domain): update_positions refuses, replan rebuilds the
    decomposition at the new coordinates (frames and reciprocal space
    re-applied), and the step equals the single engine there."""
    from oracle import frames as fr
    from paper_1906_01211_b200 import dd
    s = mdg.water_box(1728, 37.26, 9, "amoeba")
    frame, za, xa = fr.water_frames(s.molecule)
    frames = (frame, za, xa, np.asarray(s.dipole), np.asarray(s.quadrupole))
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-6, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    recip = ((40, 40, 40), 5)
    L = s.box[0]
    mol = np.asarray(s.molecule)
    shift = np.random.default_rng(2).uniform(-3, 3, (mol.max() + 1, 3))[mol]
    x = np.mod(np.asarray(s.x) + shift[:, 0], L)
    y = np.mod(np.asarray(s.y) + shift[:, 1], L)
    z = np.mod(np.asarray(s.z) + shift[:, 2], L)
    s2 = mdg.water_box(1728, 37.26, 9, "amoeba")
    s2.x, s2.y, s2.z = x, y, z
    g = dd.DomainGroup(s, 2, HALO, backend="local", list_cutoff=11.0)
    try:
        g.upload_frames(*frames)
        g.set_ewald_recip(*recip)
        g.amoeba_step(g.build_lists(lists), p)
        owned_before = [d.plan.owned.copy() for d in g.domains]
        with pytest.raises(dd.HaloStale):
            g.update_positions(x, y, z)
        g.replan(s2)
        assert any(not np.array_equal(d.plan.owned, o) for d, o in zip(g.domains, owned_before))
        assert g.check_halo(s2)
        g.amoeba_step(g.build_lists(lists), p)
        en, _, it, _ = g.energies()
        ids, f = g.owned_forces()
    finally:
        g.close()
    en0, _, it0, f0, _ = single(mdg, s2, p, frames, recip)
    F = np.zeros_like(f0)
    F[ids] = f
    assert np.abs(F - f0).max() <= 1e-8 * np.sqrt(np.mean(f0 ** 2))
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert abs(it - it0) <= 1
