"""Spatial domain decomposition over 1/2/4/8 GPUs.

One process (context) per GPU. The orthorhombic box is split on a process
grid (1x1x1, 2x1x1, 2x2x1, 2x2x2, ...); a rank OWNS the molecules whose anchor
site (the first site of the molecule, the water oxygen) lies in its slab, so
exclusions and the Halgren reduction parent stay local. Its HALO is every
other molecule with a site within `halo_width` (list cutoff + intramolecular
extent) of the slab, periodic images included. Each rank evaluates the rows
of its owned sites (owned-owned pairs once with atomic partner updates, pairs
with a halo partner in the owned row only, energy weight 1/2), so its owned
forces, fields and dipoles are complete from owned + halo data: there is no
force return. Per step
the halo coordinates are refreshed; inside the PCG solve the halo of mu (once)
and of the search direction p (every iteration) is exchanged and the CG
scalars are all-reduced (mdg_set_comm hooks, called from the C++ solver), so
every rank takes identical CG steps. Energies and virials are summed over
ranks once per step.

The plan is computed identically on every rank from the global coordinates;
send/recv lists are ordered by global site index so both sides agree.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import mdvec as M

VEC_POS, VEC_MU, VEC_P, VEC_FORCE, VEC_TORQUE, VEC_EPERM = range(6)


# ------------------------------------------------------------------ decomposition
def process_grid(size: int) -> tuple:
    """1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2; others: greedy factors."""
    dims = [1, 1, 1]
    k, a = size, 0
    f = 2
    while k > 1:
        while k % f:
            f += 1
        dims[a % 3] *= f
        k //= f
        a += 1
    return tuple(dims)


def domain_index(x, y, z, box, dims) -> np.ndarray:
    ix = np.minimum((np.asarray(x) / box[0] * dims[0]).astype(np.int64), dims[0] - 1)
    iy = np.minimum((np.asarray(y) / box[1] * dims[1]).astype(np.int64), dims[1] - 1)
    iz = np.minimum((np.asarray(z) / box[2] * dims[2]).astype(np.int64), dims[2] - 1)
    return (ix * dims[1] + iy) * dims[2] + iz


def _axis_gap(c, lo, hi, L):
    """Periodic distance from coordinates c to the interval [lo, hi) on a circle."""
    inside = (c >= lo) & (c < hi)
    d1 = np.mod(lo - c, L)
    d2 = np.mod(c - hi, L)
    return np.where(inside, 0.0, np.minimum(d1, d2))


@dataclass
class Plan:
    rank: int
    size: int
    dims: tuple
    owned: np.ndarray            # global site ids, ascending
    halo: np.ndarray             # global site ids, ascending
    send: dict = field(default_factory=dict)   # peer -> local ids of my owned sites
    recv: dict = field(default_factory=dict)   # peer -> local ids of my halo sites

    @property
    def local(self) -> np.ndarray:
        return np.concatenate([self.owned, self.halo])

    @property
    def n_owned(self) -> int:
        return int(len(self.owned))


def build_plans(x, y, z, molecule, box, size: int, halo_width: float):
    """Every rank's plan (identical on all ranks)."""
    box = tuple(map(float, box))
    dims = process_grid(size)
    n = len(x)
    mol = np.asarray(molecule)
    # anchor = first site of each molecule
    order = np.arange(n)
    first = np.full(mol.max() + 1, n, np.int64)
    np.minimum.at(first, mol, order)
    anchor = first[mol]
    dom_site = domain_index(x, y, z, box, dims)
    owner = dom_site[anchor]  # owner rank of every site (by molecule)
    pos = np.stack([np.asarray(x), np.asarray(y), np.asarray(z)], 1)
    owned = [np.nonzero(owner == r)[0] for r in range(size)]
    halos = []
    for r in range(size):
        ix, rem = divmod(r, dims[1] * dims[2])
        iy, iz = divmod(rem, dims[2])
        lo = np.array([ix, iy, iz], float) * np.array(box) / np.array(dims)
        hi = (np.array([ix, iy, iz], float) + 1) * np.array(box) / np.array(dims)
        g = np.sqrt(sum(_axis_gap(pos[:, a], lo[a], hi[a], box[a]) ** 2 for a in range(3)))
        near_mol = np.unique(mol[(g <= halo_width) & (owner != r)])
        halos.append(np.nonzero(np.isin(mol, near_mol) & (owner != r))[0])
    plans = []
    for r in range(size):
        p = Plan(r, size, dims, owned[r], halos[r])
        loc = {int(g): k for k, g in enumerate(p.local)}
        for q in range(size):
            if q == r:
                continue
            # what q needs from me: my owned sites in q's halo
            s = np.intersect1d(owned[r], halos[q], assume_unique=True)
            if len(s):
                p.send[q] = np.array([loc[int(g)] for g in s], np.int32)
            # what I need from q: q's owned sites in my halo
            t = np.intersect1d(owned[q], halos[r], assume_unique=True)
            if len(t):
                p.recv[q] = np.array([loc[int(g)] for g in t], np.int32)
        plans.append(p)
    return plans


def local_system(s, plan: Plan):
    """The rank's ParticleSystem in local order (owned, then halo)."""
    idx = plan.local
    inv = {int(g): k for k, g in enumerate(idx)}
    kw = {}
    for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
              "polarizability"):
        kw[k] = np.ascontiguousarray(np.asarray(getattr(s, k))[idx])
    mol = None if getattr(s, "molecule", None) is None else np.asarray(s.molecule)[idx]
    dip = None if getattr(s, "dipole", None) is None else np.asarray(s.dipole)[idx]
    quad = None if getattr(s, "quadrupole", None) is None else np.asarray(s.quadrupole)[idx]
    par = fac = None
    if getattr(s, "hred_parent", None) is not None:
        par = np.array([inv[int(g)] for g in np.asarray(s.hred_parent)[idx]], np.int32)
        fac = np.asarray(s.hred_factor)[idx]
    return M.ParticleSystem(tuple(s.box), molecule=mol, dipole=dip, quadrupole=quad,
                            hred_parent=par, hred_factor=fac, **kw)


# ------------------------------------------------------------------ communicators
class TorchComm:
    """torch.distributed: NCCL (device buffers) or gloo (host buffers)."""

    def __init__(self, device: int | None = None, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        self.cuda = dist.get_backend(group) == "nccl"
        self.device = torch.device(f"cuda:{device}") if self.cuda else torch.device("cpu")
        if self.cuda:
            # create the NCCL communicator with a collective every rank joins
            # (batched point-to-point must not be the group's first call)
            self.allreduce(np.zeros(1))

    def exchange(self, sends: dict, recv_counts: dict) -> dict:
        """sends: peer -> float64 buffer; returns peer -> received buffer.
        All receives and sends go out as one batch (ncclGroupStart/End under
        NCCL): two ranks that each post recv-then-send on the shared pair
        stream would otherwise wait on each other."""
        t, dist = self.torch, self.dist
        ops, out = [], {}
        for q, n in recv_counts.items():
            out[q] = t.empty(n, dtype=t.float64, device=self.device)
            ops.append(dist.P2POp(dist.irecv, out[q], q, group=self.group))
        for q, buf in sends.items():
            tb = buf if isinstance(buf, t.Tensor) else t.from_numpy(np.ascontiguousarray(buf))
            ops.append(dist.P2POp(dist.isend, tb.to(self.device), q, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if self.cuda:
            t.cuda.synchronize(self.device)
        return out

    def allreduce(self, vals: np.ndarray) -> np.ndarray:
        t = self.torch
        buf = t.from_numpy(np.array(vals, np.float64)).to(self.device)
        self.dist.all_reduce(buf, group=self.group)
        return buf.cpu().numpy()


class LocalComm:
    """In-process domains (one thread each), e.g. several contexts on one GPU
    in a test: a mailbox plus barriers. Sums are formed in rank order."""

    class _Shared:
        def __init__(self, size):
            self.size = size
            self.box = {}
            self.red = [None] * size
            self.barrier = threading.Barrier(size)

    def __init__(self, shared, rank):
        self.s, self.rank, self.size = shared, rank, shared.size
        self.cuda = False

    @classmethod
    def group(cls, size):
        sh = cls._Shared(size)
        return [cls(sh, r) for r in range(size)]

    def exchange(self, sends, recv_counts):
        for q, buf in sends.items():
            self.s.box[(self.rank, q)] = np.array(buf, np.float64)
        self.s.barrier.wait()
        out = {q: self.s.box[(q, self.rank)] for q in recv_counts}
        self.s.barrier.wait()
        for q in sends:
            self.s.box.pop((self.rank, q), None)
        return out

    def allreduce(self, vals):
        self.s.red[self.rank] = np.array(vals, np.float64)
        self.s.barrier.wait()
        tot = np.sum(np.stack(self.s.red), 0)
        self.s.barrier.wait()
        return tot


# ------------------------------------------------------------------ the rank engine
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)


class DDEngine:
    """One rank: an Engine over owned + halo sites with the comm hooks installed."""

    def __init__(self, s, comm, device: int, halo_width: float, plans=None):
        self.comm = comm
        self.plans = plans or build_plans(s.x, s.y, s.z, s.molecule, s.box, comm.size,
                                          halo_width)
        self.plan = self.plans[comm.rank]
        self.n_global = len(s.x)
        self.local = local_system(s, self.plan)
        self.eng = M.Engine(len(self.plan.local), device=device)
        self._upload()
        self._ex = EXCHANGE_FN(self._exchange_cb)
        self._ar = ALLREDUCE_FN(self._allreduce_cb)
        if comm.size > 1:
            M.check(self.eng.lib.mdg_set_comm(self.eng.ctx, C.cast(self._ex, C.c_void_p),
                                              C.cast(self._ar, C.c_void_p), None))
        self.recv_counts = {q: 3 * len(v) for q, v in self.plan.recv.items()}
        self._dev_idx = {}
        self.error = None

    def _upload(self):
        L = self.local
        arrs = [M._f64(getattr(L, k)) for k in ("x", "y", "z", "charge", "lj_sigma",
                                                 "lj_epsilon", "hal_r0", "hal_epsilon",
                                                 "polarizability")]
        self._keep = arrs
        M.check(self.eng.lib.mdg_system_upload_owned(
            self.eng.ctx, len(arrs[0]), self.plan.n_owned, self.n_global, *map(float, L.box),
            *(M._p(a) for a in arrs)))
        self.eng.n = len(arrs[0])
        self.eng.box = tuple(map(float, L.box))
        self.eng.upload_topology(L.molecule, L.hred_parent, L.hred_factor)
        if L.dipole is not None or L.quadrupole is not None:
            self.eng.upload_multipoles(L.dipole, L.quadrupole)

    def upload_frames(self, frame, zatom, xatom, dipole, quadrupole):
        """Local multipole frames (global arrays, global site ids): the
        rank's owned + halo sites with their frame atoms mapped to local
        ids (frame atoms belong to the same molecule, so they are local)."""
        idx = self.plan.local
        inv = {int(g): k for k, g in enumerate(idx)}
        fr = np.asarray(frame)[idx]
        za = np.array([inv[int(g)] if f else 0 for g, f in zip(np.asarray(zatom)[idx], fr)],
                      np.int32)
        xa = np.array([inv[int(g)] if f else 0 for g, f in zip(np.asarray(xatom)[idx], fr)],
                      np.int32)
        self.eng.upload_frames(fr, za, xa, np.asarray(dipole)[idx], np.asarray(quadrupole)[idx])

    # ---- halo traffic
    def exchange(self, vec_id: int):
        if self.comm.size == 1:
            return
        if getattr(self.comm, "cuda", False):
            self._exchange_dev(vec_id)
            return
        sends = {q: self.eng.vec_pack(vec_id, idx) for q, idx in self.plan.send.items()}
        recvs = self.comm.exchange(sends, self.recv_counts)
        for q, buf in recvs.items():
            self.eng.vec_unpack(vec_id, self.plan.recv[q], np.asarray(buf, np.float64))

    def _exchange_dev(self, vec_id: int):
        torch = self.comm.torch
        dev = self.comm.device
        if not self._dev_idx:
            for tag, d in (("s", self.plan.send), ("r", self.plan.recv)):
                for q, idx in d.items():
                    self._dev_idx[(tag, q)] = torch.from_numpy(idx).to(dev)
        sends = {}
        for q, idx in self.plan.send.items():
            buf = torch.empty(3 * len(idx), dtype=torch.float64, device=dev)
            M.check(self.eng.lib.mdg_vec_pack_dev(
                self.eng.ctx, vec_id, C.c_void_p(self._dev_idx[("s", q)].data_ptr()), len(idx),
                C.c_void_p(buf.data_ptr())))
            sends[q] = buf
        recvs = self.comm.exchange(sends, self.recv_counts)
        for q, buf in recvs.items():
            M.check(self.eng.lib.mdg_vec_unpack_dev(
                self.eng.ctx, vec_id, C.c_void_p(self._dev_idx[("r", q)].data_ptr()),
                len(self.plan.recv[q]), C.c_void_p(buf.data_ptr())))

    def _exchange_cb(self, user, vec_id):
        try:
            self.exchange(vec_id)
            return 0
        except Exception as e:  # surfaced as MDG_COMM by the solver
            self.error = e
            return 1

    def _allreduce_cb(self, user, vals, n):
        try:
            arr = np.ctypeslib.as_array(vals, (n,))
            arr[:] = self.comm.allreduce(arr)
            return 0
        except Exception as e:
            self.error = e
            return 1

    # ---- step
    def build_lists(self, lists):
        """lists: [(cutoff, list_id, sites), ...] -- rows for owned sites."""
        return {lid: self.eng.build_neighbor_table(cut, list_id=lid, sites=sites)
                for cut, lid, sites in lists}

    def update_positions(self, x, y, z):
        """New global coordinates: owned from the caller, halo refreshed by exchange."""
        own = self.plan.owned
        n = len(self.plan.local)
        lx = np.zeros(n)
        ly = np.zeros(n)
        lz = np.zeros(n)
        lx[: len(own)], ly[: len(own)], lz[: len(own)] = x[own], y[own], z[own]
        lx[len(own):] = np.asarray(x)[self.plan.halo]  # placeholder, overwritten below
        ly[len(own):] = np.asarray(y)[self.plan.halo]
        lz[len(own):] = np.asarray(z)[self.plan.halo]
        self.eng.upload_positions(lx, ly, lz)
        self.exchange(VEC_POS)

    def amoeba_step(self, tables, params):
        vdw = tables.get(1, tables[0])
        try:
            self.eng.amoeba_step(vdw, tables[0], params)
        finally:
            if self.error is not None:
                raise self.error

    def charmm_step(self, tables, params):
        self.eng.charmm_step(tables[0], params)

    def energies(self):
        """Global energies and virial (sum over ranks) and the PCG record."""
        e, w, it, rms = self.eng.fetch_energies()
        tot = self.comm.allreduce(np.concatenate([e, w.reshape(-1)])) if self.comm.size > 1 \
            else np.concatenate([e, w.reshape(-1)])
        return tot[:4], tot[4:].reshape(3, 3), it, rms

    def owned_forces(self):
        """(global ids, forces) of the owned sites."""
        f = self.eng.fetch_forces()
        return self.plan.owned, f[: self.plan.n_owned]

    def owned_dipoles(self):
        mu = self.eng.fetch_dipoles()
        return self.plan.owned, mu[: self.plan.n_owned]

    def check_halo(self, s) -> bool:
        """Self-check of the exchange path: refresh the halo coordinates and
        compare them with the global fixture every rank holds."""
        if not len(self.plan.halo):
            return True
        n_own = self.plan.n_owned
        halo_local = np.arange(n_own, n_own + len(self.plan.halo), dtype=np.int32)
        # scramble the halo, then let the exchange restore it
        self.eng.vec_unpack(VEC_POS, halo_local, np.zeros(3 * len(halo_local)))
        self.exchange(VEC_POS)
        got = self.eng.vec_pack(VEC_POS, halo_local).reshape(-1, 3)
        want = np.stack([np.asarray(s.x), np.asarray(s.y), np.asarray(s.z)], 1)[self.plan.halo]
        return bool(np.array_equal(got, want))

    def close(self):
        self.eng.lib.mdg_set_comm(self.eng.ctx, None, None, None)
        self.eng.close()
