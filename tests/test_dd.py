"""Spatial domain decomposition.

CPU: the decomposition plan (ownership, halo completeness, send/recv
symmetry) and a world-size-2 gloo run in which
every rank builds its NCCL halo arguments with the product code
(dd.nccl_halo_args) and checks them against its peer's over gloo, then runs
the multi-domain solve protocol of csrc/polar.cu run_pcg_multi (halo refresh
of the direction, three summed CG scalars per iteration) with the oracle's
kernels on its local system, against the single-domain oracle. The device
runtime itself (csrc/group.cu, LOCAL and NCCL backends) is exercised on the
GPU in tests/test_gpu_dd.py.
"""
import os
import socket

import numpy as np
import pytest

from conftest import to_oracle_system

HALO = 10.5  # list 9 A + intramolecular extent + margin


def water(mdg, n_mol=512, box=24.8, seed=3):
    return mdg.water_box(n_mol, box, seed, "amoeba")


@pytest.mark.parametrize("size", [2, 4, 8])
def test_plan_partition_and_halo(mdg, size):
    from paper_1906_01211_b200 import dd
    s = water(mdg, 1000, 31.04)
    plans = dd.build_plans(s.x, s.y, s.z, s.molecule, s.box, size, HALO)
    assert dd.process_grid(size) == {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[size]
    owned = np.concatenate([p.owned for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(s.n_sites))  # a partition
    mol = np.asarray(s.molecule)
    for p in plans:
        # whole molecules only
        assert set(np.unique(mol[p.owned])) == set(mol[p.owned])
        assert not np.isin(mol[p.halo], mol[p.owned]).any()
        # completeness: every site within 9 A (minimum image) of an owned site is local
        loc = np.zeros(s.n_sites, bool)
        loc[p.local] = True
        P = np.stack([s.x, s.y, s.z], 1)
        L = np.array(s.box)
        for i in p.owned[::37]:
            d = P - P[i]
            d -= L * np.round(d / L)
            near = np.nonzero(np.sum(d * d, 1) <= 9.0 ** 2)[0]
            assert loc[near].all()
    # send/recv symmetry, same global ids in the same order
    for r, p in enumerate(plans):
        for q, idx in p.recv.items():
            assert r in plans[q].send
            g_recv = p.local[idx]
            g_send = plans[q].local[plans[q].send[r]]
            assert np.array_equal(g_recv, g_send)


# ---------------------------------------------------------------- gloo world 2
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, size, port, out_dir):
    import torch.distributed as dist

    import paper_1906_01211_b200 as mdg
    from oracle.oracle import Oracle
    from paper_1906_01211_b200 import dd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import torch
        o = Oracle()
        comm = _GlooComm(dist, torch)
        s = water(mdg)
        plans = dd.build_plans(s.x, s.y, s.z, s.molecule, s.box, size, HALO)
        p = plans[rank]
        # the product's NCCL halo arguments agree with the peer's (global ids, order)
        peers, sc, ss, rc, rs = dd.nccl_halo_args(p)
        mine = {"send": {}, "recv": {}}
        so = ro = 0
        for k, q in enumerate(peers):
            mine["send"][int(q)] = p.local[ss[so:so + sc[k]]].tolist()
            mine["recv"][int(q)] = p.local[rs[ro:ro + rc[k]]].tolist()
            so += sc[k]
            ro += rc[k]
        allargs = [None] * size
        dist.all_gather_object(allargs, mine)
        for q in range(size):
            if q != rank:
                assert allargs[q]["send"].get(rank, []) == mine["recv"].get(q, [])
                assert allargs[q]["recv"].get(rank, []) == mine["send"].get(q, [])
        loc = to_oracle_system(dd.local_system(s, p))
        n_own = p.n_owned
        alpha, cut, thole = 0.5446, 7.0, 0.39

        # pair forces on owned rows + owned-row energy 1/2 (E_all + E_own - E_halo)
        t_all = o.build_table(loc, 9.0)
        f, e_all, _ = o.ewald_real(loc, t_all, alpha, cut, 1.0, exclude=True)
        own_sys = loc.copy()
        halo_sys = loc.copy()
        for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
                  "polarizability", "molecule", "dipole", "quadrupole"):
            a = getattr(loc, k)
            setattr(own_sys, k, None if a is None else a[:n_own])
            setattr(halo_sys, k, None if a is None else a[n_own:])
        e_own = o.ewald_real(own_sys, o.build_table(own_sys, 9.0), alpha, cut, 1.0, True)[1]
        e_halo = (o.ewald_real(halo_sys, o.build_table(halo_sys, 9.0), alpha, cut, 1.0, True)[1]
                  if halo_sys.n else 0.0)
        e_rank = 0.5 * (e_all + e_own - e_halo)
        e_tot = comm.allreduce([e_rank])[0]
        fg = np.zeros((s.n_sites, 3))
        fg[p.owned] = f[:n_own]
        fg = comm.allreduce(fg.reshape(-1)).reshape(-1, 3)

        # multi-domain PCG: the protocol of run_pcg_multi (halo of mu / p before
        # each mat-vec, r.z / p.q / (r.z, |dmu|^2) summed over the domains)
        E = o.perm_field_ewald(loc, t_all, alpha, cut, thole, exclude=True)
        pol = loc.polarizability[:, None]

        def exchange(v):
            sends = {q: v[idx].reshape(-1) for q, idx in p.send.items()}
            recvs = comm.exchange(sends, {q: 3 * len(i) for q, i in p.recv.items()})
            for q, buf in recvs.items():
                v[p.recv[q]] = np.asarray(buf).reshape(-1, 3)

        def T(v):
            return o.tmatvec_ewald(loc, t_all, alpha, cut, thole, v)

        mu = np.zeros_like(E)
        mu[:n_own] = pol[:n_own] * E[:n_own]
        exchange(mu)
        tm = T(mu)
        r = E - (mu / pol - tm)
        r[n_own:] = 0
        z = pol * r
        pvec = z.copy()
        rz = comm.allreduce([np.sum(r[:n_own] * z[:n_own])])[0]
        it = 0
        for it in range(1, 100):
            exchange(pvec)
            q = pvec / pol - T(pvec)
            pq = comm.allreduce([np.sum(pvec[:n_own] * q[:n_own])])[0]
            a = rz / pq
            mu[:n_own] += a * pvec[:n_own]
            r[:n_own] -= a * q[:n_own]
            z = pol * r
            rzn, ds = comm.allreduce([np.sum(r[:n_own] * z[:n_own]),
                                      np.sum((a * pvec[:n_own]) ** 2)])
            rms = np.sqrt(ds / s.n_sites) * mdg.DEBYE
            if rms < 1e-5:
                break
            pvec[:n_own] = z[:n_own] + (rzn / rz) * pvec[:n_own]
            rz = rzn
        mug = np.zeros((s.n_sites, 3))
        mug[p.owned] = mu[:n_own]
        mug = comm.allreduce(mug.reshape(-1)).reshape(-1, 3)
        if rank == 0:
            np.savez(os.path.join(out_dir, "dd.npz"), f=fg, e=e_tot, mu=mug, it=it)
    finally:
        dist.destroy_process_group()


class _GlooComm:
    """Host-buffer halo exchange + all-reduce over gloo (test transport)."""

    def __init__(self, dist, torch):
        self.dist, self.torch = dist, torch

    def exchange(self, sends, recv_counts):
        t, dist = self.torch, self.dist
        ops, out = [], {}
        for q, n in recv_counts.items():
            out[q] = t.empty(n, dtype=t.float64)
            ops.append(dist.P2POp(dist.irecv, out[q], q))
        for q, buf in sends.items():
            ops.append(dist.P2POp(dist.isend, t.from_numpy(np.ascontiguousarray(buf)), q))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return {q: v.numpy() for q, v in out.items()}

    def allreduce(self, vals):
        buf = self.torch.from_numpy(np.array(vals, np.float64))
        self.dist.all_reduce(buf)
        return buf.numpy()


def test_gloo_world2_matches_single_domain(tmp_path, oracle, mdg):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = np.load(os.path.join(tmp_path, "dd.npz"))
    s = water(mdg)
    so = to_oracle_system(s)
    t = oracle.build_table(so, 9.0)
    f, e, _ = oracle.ewald_real(so, t, 0.5446, 7.0, 1.0, exclude=True)
    assert float(got["e"]) == pytest.approx(e, rel=1e-10)
    assert np.abs(got["f"] - f).max() <= 1e-10 * np.abs(f).max()
    E = oracle.perm_field_ewald(so, t, 0.5446, 7.0, 0.39, exclude=True)
    mu, it, _ = oracle.pcg(so, t, 0.5446, 7.0, 0.39, E, 1e-5, 100)
    assert abs(int(got["it"]) - it) <= 1
    d = np.sqrt(np.mean(np.sum((got["mu"] - mu) ** 2, 1))) * mdg.DEBYE
    assert d < 1e-5
