"""Spatial domain decomposition over 1/2/4/8 GPUs.

The orthorhombic box is split on a process grid (1x1x1, 2x1x1, 2x2x1,
2x2x2, ...); a domain OWNS the molecules whose anchor site (the first site of
the molecule, the water oxygen) lies in its subdomain, so exclusions and the
Halgren reduction parent stay local. Its HALO is every other molecule with a
site within `halo_width` (list cutoff + intramolecular extent) of the
subdomain, periodic images included. Each domain evaluates the rows of its
owned sites (owned-owned pairs once with atomic partner updates, pairs with a
halo partner in the owned row only, energy weight 1/2), so its owned forces,
fields and dipoles are complete from owned + halo data: there is no force
return (DESIGN.md 7 gives the cost comparison with a half-shell halo).

This module builds the plan (identical on every rank, from the global
coordinates; send/recv lists ordered by global site id so both sides agree)
and drives the C++ group runtime (csrc/group.cu, include/mdg.h mdg_group_*):
per step the halo coordinates are refreshed; inside the PCG solve the halo of
the search direction is exchanged and the CG scalars are summed on the device
every iteration, with no host round trip. Two backends: LOCAL (every domain
in this process on one device: the single-GPU emulation of N ranks) and NCCL
(one domain per torch.distributed rank / GPU).
"""
from __future__ import annotations

import ctypes as C
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


# ------------------------------------------------------------------ the runtime
class Domain:
    """One domain: an Engine over its owned + halo sites (local order =
    plan.local: owned first, then halo, each ascending in global id)."""

    def __init__(self, s, plan: Plan, n_global: int, device: int):
        self.plan = plan
        self.local = local_system(s, plan)
        self.eng = M.Engine(len(plan.local), device=device)
        L = self.local
        arrs = [M._f64(getattr(L, k)) for k in ("x", "y", "z", "charge", "lj_sigma",
                                                 "lj_epsilon", "hal_r0", "hal_epsilon",
                                                 "polarizability")]
        self._keep = arrs
        M.check(self.eng.lib.mdg_system_upload_owned(
            self.eng.ctx, len(arrs[0]), plan.n_owned, n_global, *map(float, L.box),
            *(M._p(a) for a in arrs)))
        self.eng.n = len(arrs[0])
        self.eng.box = tuple(map(float, L.box))
        self.eng.upload_topology(L.molecule, L.hred_parent, L.hred_factor)
        if L.dipole is not None or L.quadrupole is not None:
            self.eng.upload_multipoles(L.dipole, L.quadrupole)

    def upload_frames(self, frame, zatom, xatom, dipole, quadrupole):
        """Local multipole frames (global arrays, global site ids) mapped to
        local ids (frame atoms belong to the same molecule, so are local)."""
        idx = self.plan.local
        inv = np.full(int(max(idx.max(), np.max(zatom), np.max(xatom))) + 1, -1, np.int64)
        inv[idx] = np.arange(len(idx))
        fr = np.asarray(frame)[idx]
        za = np.where(fr != 0, inv[np.asarray(zatom)[idx]], 0).astype(np.int32)
        xa = np.where(fr != 0, inv[np.asarray(xatom)[idx]], 0).astype(np.int32)
        self.eng.upload_frames(fr, za, xa, np.asarray(dipole)[idx], np.asarray(quadrupole)[idx])


def nccl_halo_args(p: Plan):
    """Arguments of mdg_group_set_halo_nccl for one rank's plan: peer ranks
    (ascending), per-peer send / recv counts, and the caller-order local
    indices concatenated per peer. Rank r's sends to q and q's receives from r
    list the same global sites in the same (ascending global id) order."""
    peers = sorted(set(p.send) | set(p.recv))
    sc = np.array([len(p.send.get(q, ())) for q in peers], np.int64)
    rc = np.array([len(p.recv.get(q, ())) for q in peers], np.int64)
    ss = np.concatenate([p.send[q] for q in peers if q in p.send] or
                        [np.zeros(0, np.int32)]).astype(np.int32)
    rs = np.concatenate([p.recv[q] for q in peers if q in p.recv] or
                        [np.zeros(0, np.int32)]).astype(np.int32)
    return np.array(peers, np.int32), sc, ss, rc, rs


class HaloStale(RuntimeError):
    """Sites moved farther than the halo margin allows since the plan was built."""


class DomainGroup:
    """The decomposed system's runtime over the C++ group (mdg_group_*).

    backend "local": every domain in this process on `device` (one context
    per domain, one shared stream) -- N ranks emulated on one GPU.
    backend "nccl": this rank's domain only; `rank`/`size` of the
    torch.distributed default group, which also carries the NCCL unique id.
    overlap: interior/halo overlap in the PCG (None: the engine's default,
    on for NCCL, off for LOCAL).
    """

    def __init__(self, s, size: int, halo_width: float, device: int = 0, backend: str = "local",
                 rank: int = 0, plans=None, list_cutoff: float | None = None,
                 overlap: bool | None = None):
        self._args = dict(size=size, halo_width=halo_width, device=device, backend=backend,
                          rank=rank, list_cutoff=list_cutoff, overlap=overlap)
        self._frames = self._recip = None
        self.lib = M.load_library()
        self.backend, self.size, self.rank = backend, size, rank
        self.halo_width = float(halo_width)
        self.n_global = len(s.x)
        self.box = np.asarray(s.box, float)
        self.plans = plans or build_plans(s.x, s.y, s.z, s.molecule, s.box, size, halo_width)
        # sites may move (halo_width - list cutoff - 1 A intramolecular extent) / 2
        # before the halo can miss a pair (update_positions checks)
        lc = list_cutoff if list_cutoff is not None else halo_width - 1.5
        self.margin = max(0.0, (self.halo_width - lc - 1.0) / 2.0)
        mine = range(size) if backend == "local" else [rank]
        self.domains = [Domain(s, self.plans[r], self.n_global, device) for r in mine]
        self.g = C.c_void_p()
        if backend == "local":
            ctxs = (C.c_void_p * len(self.domains))(*[d.eng.ctx.value for d in self.domains])
            M.check(self.lib.mdg_group_create_local(C.byref(self.g), len(self.domains), ctxs,
                                                    self.n_global))
            self._set_halo_local()
        elif backend == "nccl":
            import torch.distributed as dist
            uid = C.create_string_buffer(128)
            if rank == 0:
                M.check(self.lib.mdg_nccl_unique_id(uid))
            obj = [bytes(uid.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = C.create_string_buffer(obj[0], 128)
            M.check(self.lib.mdg_group_create_nccl(C.byref(self.g), self.domains[0].eng.ctx,
                                                   rank, size, uid, self.n_global))
            self._set_halo_nccl()
        else:
            raise ValueError(f"unknown backend {backend!r}")
        if overlap is not None:  # interior/halo overlap (mdg.h mdg_group_set_overlap)
            M.check(self.lib.mdg_group_set_overlap(self.g, int(bool(overlap))))
        M.check(self.lib.mdg_group_set_reference(self.g))

    # ---- halo plans
    def _set_halo_local(self):
        owner = np.empty(self.n_global, np.int32)
        where = np.empty(self.n_global, np.int32)  # caller-order local index in the owner
        for r, p in enumerate(self.plans):
            owner[p.owned] = r
            where[p.owned] = np.arange(p.n_owned, dtype=np.int32)
        for d, p in enumerate(self.plans):
            halo_local = np.arange(p.n_owned, p.n_owned + len(p.halo), dtype=np.int32)
            src_dom = np.ascontiguousarray(owner[p.halo])
            src_site = np.ascontiguousarray(where[p.halo])
            M.check(self.lib.mdg_group_set_halo_local(
                self.g, d, len(p.halo), M._p(halo_local, M._ip), M._p(src_dom, M._ip),
                M._p(src_site, M._ip)))

    def _set_halo_nccl(self):
        peers, sc, ss, rc, rs = nccl_halo_args(self.plans[self.rank])
        M.check(self.lib.mdg_group_set_halo_nccl(
            self.g, len(peers), M._p(peers, M._ip), M._p(sc, M._i64p), M._p(ss, M._ip),
            M._p(rc, M._i64p), M._p(rs, M._ip)))

    # ---- per step
    def exchange(self, vec_id: int):
        M.check(self.lib.mdg_group_exchange(self.g, vec_id))

    def upload_frames(self, frame, zatom, xatom, dipole, quadrupole):
        self._frames = (frame, zatom, xatom, dipole, quadrupole)
        for d in self.domains:
            d.upload_frames(frame, zatom, xatom, dipole, quadrupole)

    def replan(self, s):
        """Molecule migration by re-planning: after sites moved past the
        halo margin (HaloStale), rebuild the decomposition from the global
        system `s` at its current coordinates -- ownership by the anchor
        site's subdomain, halos, contexts, the group -- and re-apply the
        frames and the reciprocal-space grid. Collective over the ranks of an
        NCCL group (every rank passes the same global coordinates). The
        neighbour lists are rebuilt by the caller (build_lists)."""
        frames, recip = self._frames, self._recip
        self.close()
        self.__init__(s, **self._args)
        if frames is not None:
            self.upload_frames(*frames)
        if recip is not None:
            self.set_ewald_recip(*recip)

    def set_ewald_recip(self, grid=(0, 0, 0), order: int = 6):
        """Reciprocal-space Ewald in the decomposed AMOEBA step (every domain
        the same grid): each domain spreads its owned sites, the grids are
        summed over the domains (one device: a kernel; NCCL: an all-reduce),
        the sum is transformed once per device and every domain gathers its
        owned sites -- a replicated grid, not a distributed FFT."""
        self._recip = (grid, order)
        for d in self.domains:
            d.eng.set_ewald_recip(grid, order)

    def build_lists(self, lists):
        """lists: [(cutoff, list_id, sites), ...]: every local domain builds the
        rows of its owned sites (candidates: owned + halo)."""
        for d in self.domains:
            for cut, lid, sites in lists:
                d.eng.build_neighbor_table(cut, list_id=lid, sites=sites)
        return {lid: lid for _, lid, _ in lists}

    def update_positions(self, x, y, z):
        """New global coordinates: each domain uploads its local sites' (the
        halo part is then refreshed from the owners by the group exchange).
        Raises HaloStale when a site has moved past half the halo margin since
        the plan was built (checked on the device, max over all domains)."""
        for dom in self.domains:
            # owned coordinates only, gathered into page-locked buffers (DMA'd
            # without staging); the halo comes from the owners below
            own = dom.plan.owned
            if getattr(dom, "_xyz", None) is None:
                dom._xyz = M.host_array((3, len(own)))
            for a, v in enumerate((x, y, z)):
                np.take(np.asarray(v, np.float64), own, out=dom._xyz[a])
            dom.eng.upload_positions_owned(dom._xyz[0], dom._xyz[1], dom._xyz[2])
        moved = self.max_displacement()
        if moved > self.margin:
            raise HaloStale(f"a site moved {moved:.3f} A since the plan was built "
                            f"(margin {self.margin:.3f} A): rebuild the plan")
        self.exchange(VEC_POS)

    def max_displacement(self) -> float:
        v = C.c_double()
        M.check(self.lib.mdg_group_max_displacement(self.g, C.byref(v)))
        return v.value

    def amoeba_step(self, tables, params):
        vdw = tables.get(1, tables[0])
        M.check(self.lib.mdg_group_amoeba_step(self.g, vdw, tables[0], C.byref(params)))

    def charmm_step(self, tables, params):
        M.check(self.lib.mdg_group_charmm_step(self.g, tables[0], C.byref(params)))

    def energies(self):
        """Global energies and virial (all domains, all ranks) and the PCG record."""
        e = np.zeros(4)
        w = np.zeros(9)
        it = C.c_int64()
        rms = C.c_double()
        M.check(self.lib.mdg_group_fetch_energies(self.g, M._p(e), M._p(w), C.byref(it),
                                                  C.byref(rms)))
        return e, w.reshape(3, 3), it.value, rms.value

    def owned_forces(self):
        """(global ids, forces) of the owned sites of the local domains."""
        ids = [d.plan.owned for d in self.domains]
        f = [d.eng.fetch_forces()[: d.plan.n_owned] for d in self.domains]
        return np.concatenate(ids), np.concatenate(f)

    def owned_dipoles(self):
        ids = [d.plan.owned for d in self.domains]
        mu = [d.eng.fetch_dipoles()[: d.plan.n_owned] for d in self.domains]
        return np.concatenate(ids), np.concatenate(mu)

    def check_halo(self, s) -> bool:
        """Self-check of the exchange path: scramble every local domain's halo
        coordinates, refresh them from the owners, compare with the fixture."""
        want_all = np.stack([np.asarray(s.x), np.asarray(s.y), np.asarray(s.z)], 1)
        for d in self.domains:
            p = d.plan
            if len(p.halo):
                halo_local = np.arange(p.n_owned, p.n_owned + len(p.halo), dtype=np.int32)
                d.eng.vec_unpack(VEC_POS, halo_local, np.zeros(3 * len(halo_local)))
        self.exchange(VEC_POS)
        ok = True
        for d in self.domains:
            p = d.plan
            if len(p.halo):
                halo_local = np.arange(p.n_owned, p.n_owned + len(p.halo), dtype=np.int32)
                got = d.eng.vec_pack(VEC_POS, halo_local).reshape(-1, 3)
                ok &= bool(np.array_equal(got, want_all[p.halo]))
        return ok

    def launch_count(self) -> int:
        return sum(d.eng.launch_count() for d in self.domains)

    def close(self):
        if getattr(self, "g", None) and self.g.value:
            self.lib.mdg_group_destroy(self.g)
            self.g = C.c_void_p()
        for d in getattr(self, "domains", []):
            d.eng.close()
