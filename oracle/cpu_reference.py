"""CPU reference arm / CPU baseline for bench.py (bench infrastructure only).

Times the reference's own CPU implementation of the path -- the unmodified
reference library in oracle/_ref (neighbor_build, lj, ewald_real, halgren,
tmatxb, all on its vectorised "Vec" path) -- on the box's host cores, and the
closed-form port oracle/mdo_fast.c (Vec flags) for the kernels the reference
lacks (real-space multipoles, multipole permanent field). Parallelism is the
reference's own: independent replicas per thread (`shards`,
proj/src/bench.cpp:330-360), seeds seed + s.

Bounded sample: the configs 1-4 step runs on an 8,000-molecule box (24,000
atoms, L = 62.1 A) of the same generator and density as the requested
config; per-atom cost in homogeneous water does not depend on box size
except through cache effects, which favour the CPU at the smaller size, so
the rate is an upper bound for the CPU on the larger configs.
"""
from __future__ import annotations

import os
import threading
import time

import numpy as np

from .oracle import FastPort, RefLib, System, Table, ref_isa

CONFIG_STEP = {
    # config: (n_mol, box, model, terms) for the CPU sample
    0: (1000, 31.04, "charmm", "lj+ewald"),
    1: (8000, 62.1, "amoeba", "vdw+mpole"),
    2: (8000, 62.1, "amoeba", "polar"),
    3: (8000, 62.1, "amoeba", "vdw+mpole+polar"),
    4: (8000, 62.1, "amoeba", "vdw+mpole+polar"),
}


def _to_system(ps) -> System:
    s = System(tuple(ps.box), ps.x, ps.y, ps.z, ps.charge, ps.lj_sigma, ps.lj_epsilon,
               ps.hal_r0, ps.hal_epsilon, ps.polarizability, molecule=ps.molecule,
               dipole=getattr(ps, "dipole", None), quadrupole=getattr(ps, "quadrupole", None))
    return s


class Replica:
    """One thread's system, reference handles and tables."""

    def __init__(self, config: int, seed: int, pcg_iters: int, rebuild_every: int = 20):
        from paper_1906_01211_b200.mdvec import reduce_sites_host, water_box  # host-only fixture
        n_mol, box, model, terms = CONFIG_STEP[config]
        self.terms = terms
        self.pcg_iters = pcg_iters
        self.rebuild_every = rebuild_every
        ps = water_box(n_mol, box, seed, model)
        self.n = ps.n_sites
        self.sys = _to_system(ps)
        self.ref = RefLib()
        self.port = FastPort()
        self.h_atom = self.ref.handle(self.sys)
        if model == "amoeba":
            xr, yr, zr = reduce_sites_host(ps)
            sv = self.sys.copy()
            sv.x, sv.y, sv.z = xr, yr, zr
            self.h_vdw = self.ref.handle(sv)
        self.mol = np.asarray(ps.molecule)
        self.tables = {}
        self.t_build = self.build(time_it=True)  # one rebuild, amortised per step
        self.st = self.sys.as_struct()
        self.mu = np.asarray(ps.dipole) if ps.dipole is not None else None

    def build(self, time_it=True) -> float:
        """Reference neighbor build(s) (Vec path); exclusion filtering (adapter,
        SURVEY 8(c)) is not timed."""
        t0 = time.perf_counter()
        if self.terms == "lj+ewald":
            raw = {"elec": self.h_atom.build_table(11.0)}
        else:
            raw = {"elec": self.h_atom.build_table(9.0)}
            if "vdw" in self.terms:
                raw["vdw"] = self.h_vdw.build_table(11.0)
        dt = time.perf_counter() - t0
        for k, t in raw.items():
            self.tables[k] = (t, t.filtered(self.mol))
        if "vdw" in self.tables:
            self.h_vdw.set_table(self.tables["vdw"][1])
        self.h_atom.set_table(self.tables["elec"][1])
        self.tt_f = self.tables["elec"][1].as_struct()
        self.tt_raw = self.tables["elec"][0].as_struct()
        return dt if time_it else 0.0

    def step(self) -> float:
        """One force evaluation (+1/rebuild_every of a list rebuild)."""
        t_build = self.t_build / self.rebuild_every
        t0 = time.perf_counter()
        if self.terms == "lj+ewald":
            self.h_atom.forces("lj", 9.0, vec=True)
            self.h_atom.forces("ewald_real", 9.0, 0.35, vec=True)
        if "vdw" in self.terms:
            self.h_vdw.forces("halgren", 9.0, 0.07, 0.12, vec=True)
        if "mpole" in self.terms:
            self.port.mpole(self.sys, None, 0.5446, 7.0, 332.063713, True, st=self.st,
                            tt=self.tt_f)
        if "polar" in self.terms:
            self.port.perm_field(self.sys, None, 0.5446, 7.0, 0.39, True, st=self.st,
                                 tt=self.tt_f)
            # the reference's own T mat-vec (tmatxb, Thole-only) on the unfiltered list
            self.h_atom.set_table(self.tables["elec"][0])
            mu = self.mu if self.mu is not None else np.zeros((self.n, 3))
            for _ in range(self.pcg_iters):
                self.h_atom.field("tmatxb", 7.0, 0.39, mu, vec=True)
            self.h_atom.set_table(self.tables["elec"][1])
        return time.perf_counter() - t0 + t_build


def run(config: int, threads: int, steps: int, warmup: int, seed: int = 1,
        pcg_iters: int = 10) -> dict:
    """Runs `threads` independent replicas; returns atom-steps/s (aggregate)."""
    reps = [Replica(config, seed + s, pcg_iters) for s in range(threads)]
    times = [[] for _ in range(threads)]

    def work(k):
        for _ in range(warmup):
            reps[k].step()
        for _ in range(steps):
            times[k].append(reps[k].step())

    th = [threading.Thread(target=work, args=(k,)) for k in range(threads)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    per_step = max(float(np.mean(t)) for t in times)  # slowest replica
    n = reps[0].n
    return {
        "value": threads * n / per_step,
        "unit": "atom-steps/s",
        "cores": threads,
        "s_per_step": per_step,
        "wall_s": wall,
        "n_sample_atoms": n,
        "isa": ref_isa(),
    }
