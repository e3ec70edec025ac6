"""GPU: the multi-domain product path (DDEngine over libmdg.so: owned + halo
contexts, halo exchange and all-reduce hooks inside the C++ PCG solve) with
2 and 4 domains hosted on ONE GPU -- one context and one host thread per
domain, exchanging through LocalComm -- against the single-domain engine.
(No kernel waits on another: the domains synchronise on the host.)"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HALO = 12.5  # 11 A vdW list + intramolecular extent + margin


def run_domains(mdg, s, size, params, lists, frames=None):
    from paper_1906_01211_b200 import dd
    comms = dd.LocalComm.group(size)
    plans = dd.build_plans(s.x, s.y, s.z, s.molecule, s.box, size, HALO)
    out = [None] * size
    errs = []

    def work(r):
        try:
            e = dd.DDEngine(s, comms[r], 0, HALO, plans=plans)
            if frames is not None:
                e.upload_frames(*frames)
            tables = e.build_lists(lists)
            e.amoeba_step(tables, params)
            en, w, it, rms = e.energies()
            ids, f = e.owned_forces()
            _, mu = e.owned_dipoles()
            out[r] = (ids, f, mu, en, w, it)
            e.close()
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)
            raise

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    n = s.n_sites
    F = np.zeros((n, 3))
    MU = np.zeros((n, 3))
    for ids, f, mu, *_ in out:
        F[ids] = f
        MU[ids] = mu
    return F, MU, out[0][3], out[0][4], out[0][5]


@pytest.mark.parametrize("size,polar_forces", [(2, False), (4, False), (2, True)])
def test_domains_match_single_gpu(mdg, size, polar_forces):
    s = mdg.water_box(1728, 37.26, 5, "amoeba")
    terms = (mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
             if polar_forces else 0)
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    with mdg.Engine(s.n_sites) as e:
        e.upload_system(s)
        te = e.build_neighbor_table(9.0, list_id=0)
        tv = e.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
        e.amoeba_step(tv, te, p)
        en0, w0, it0, _ = e.fetch_energies()
        f0 = e.fetch_forces()
        mu0 = e.fetch_dipoles()
    F, MU, en, w, it = run_domains(mdg, s, size, p, lists)
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert np.allclose(w, w0, rtol=1e-9, atol=1e-9 * np.abs(w0).max())
    assert abs(it - it0) <= 1
    d = np.sqrt(np.mean(np.sum((MU - mu0) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-5


def test_domains_with_local_frames(mdg):
    """Local multipole frames in the decomposed step (frame atoms mapped to
    each rank's local ids) match the single engine."""
    from oracle import frames as fr
    s = mdg.water_box(1728, 37.26, 6, "amoeba")
    frame, za, xa = fr.water_frames(s.molecule)
    frames = (frame, za, xa, np.asarray(s.dipole), np.asarray(s.quadrupole))
    terms = mdg.TERM_VDW | mdg.TERM_MPOLE | mdg.TERM_POLAR | mdg.TERM_POLAR_FORCE
    p = mdg.AmoebaParams(9.0, 0.07, 0.12, 7.0, 0.5446, mdg.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
    lists = [(9.0, 0, mdg.SITES_ATOMIC), (11.0, 1, mdg.SITES_VDW)]
    with mdg.Engine(s.n_sites) as e:
        e.upload_system(s)
        e.upload_frames(*frames)
        te = e.build_neighbor_table(9.0, list_id=0)
        tv = e.build_neighbor_table(11.0, list_id=1, sites=mdg.SITES_VDW)
        e.amoeba_step(tv, te, p)
        en0, w0, it0, _ = e.fetch_energies()
        f0 = e.fetch_forces()
    F, MU, en, w, it = run_domains(mdg, s, 2, p, lists, frames)
    rms = np.sqrt(np.mean(f0 ** 2))
    assert np.abs(F - f0).max() <= 1e-8 * rms
    for k in range(3):
        assert en[k] == pytest.approx(en0[k], rel=1e-9)
    assert abs(it - it0) <= 1
