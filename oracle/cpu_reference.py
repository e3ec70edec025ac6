"""CPU reference arm / CPU baseline for bench.py (bench infrastructure only).

Times the reference's own CPU implementation of the path -- the unmodified
reference library in oracle/_ref (neighbour build, Halgren, the Thole T
mat-vec `tmatxb`) on its vectorised "Vec" path and, beside it, its scalar
"Rel" path -- with the reference's own protocol
(proj/src/bench.cpp:259-283: warm-up runs, then repeats that time Scalar and
Vec back to back so slow phases hit both; trimmed mean, :389-396). The
multipole energy/forces and the multipole permanent field have no reference
implementation; they are timed with the builder's closed-form CPU
restatement oracle/mdo_fast.c (Vec flags) and reported separately as
"CPU restatement (not reference)". Parallelism is the reference's own:
independent replicas per thread (`shards`, proj/src/bench.cpp:330-360),
seeds seed + s.

The fixture comes from the oracle's own generator (mdo_water_generate, bit-
identical to the product's; tests/test_oracle.py), so this arm never loads
the product library.

Bounded sample: a configs 1-4 step runs on an 8,000-molecule box (24,000
atoms, L = 62.1 A) of the same generator and density. The per-atom CPU cost
of the step measured at 24k, 96k and 1M atoms is committed in
profiles/r2_cpu_cost_curve.json (scratch: oracle/cpu_cost_curve.py).
"""
from __future__ import annotations

import os
import threading
import time

import numpy as np

from .oracle import FastPort, Oracle, RefLib, ref_isa

# config: (n_mol, box, model, terms) of the CPU sample
CONFIG_STEP = {
    0: (1000, 31.04, "charmm", "lj+ewald"),
    1: (8000, 62.1, "amoeba", "vdw+mpole"),
    2: (8000, 62.1, "amoeba", "polar"),
    3: (8000, 62.1, "amoeba", "vdw+mpole+polar"),
    4: (8000, 62.1, "amoeba", "vdw+mpole+polar"),
}
# PCG mat-vecs per step: the GPU solve's iteration count on the BASELINE
# fixture (BENCH_r01.json: 8 iterations + the initial mat-vec)
GPU_PCG_MATVECS = 9


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def trimmed_mean(v) -> float:
    """proj/src/bench.cpp:389-396 (drop min and max; needs >= 3 samples)."""
    v = sorted(v)
    if len(v) < 3:
        raise ValueError("trimmed_mean: need at least 3 samples")
    return float(np.mean(v[1:-1]))


class Replica:
    """One thread's system, reference handles and tables."""

    def __init__(self, config: int, seed: int, matvecs: int = GPU_PCG_MATVECS,
                 rebuild_every: int = 20, n_mol: int | None = None, box: float | None = None,
                 scalar: bool = True):
        n_mol0, box0, model, terms = CONFIG_STEP[config]
        n_mol = n_mol or n_mol0
        box = box or box0
        self.terms = terms
        self.matvecs = matvecs
        self.rebuild_every = rebuild_every
        o = Oracle()
        s, par, fac = o.water_box(n_mol, box, seed, model)
        self.n = s.n
        self.sys = s
        self.ref = RefLib()
        self.port = FastPort()
        self.h_atom = self.ref.handle(s)
        if model == "amoeba":
            xr, yr, zr = o.reduce_sites(s, par, fac)
            sv = s.copy()
            sv.x, sv.y, sv.z = xr, yr, zr
            self.h_vdw = self.ref.handle(sv)
        self.mol = np.asarray(s.molecule)
        self.tables = {}
        self.t_build = {True: self.build(True)}
        if scalar:
            self.t_build[False] = self.build(False)
            self.build(True)  # leave the Vec tables installed
        self.st = s.as_struct()
        self.mu = np.asarray(s.dipole) if s.dipole is not None else np.zeros((self.n, 3))

    def build(self, vec: bool) -> float:
        """Reference neighbour build(s); the exclusion filtering (adapter, SURVEY
        8(c)) is not timed."""
        t0 = time.perf_counter()
        if self.terms == "lj+ewald":
            raw = {"elec": self.h_atom.build_table(11.0, vec=vec)}
        else:
            raw = {"elec": self.h_atom.build_table(9.0, vec=vec)}
            if "vdw" in self.terms:
                raw["vdw"] = self.h_vdw.build_table(11.0, vec=vec)
        dt = time.perf_counter() - t0
        for k, t in raw.items():
            self.tables[k] = (t, t.filtered(self.mol))
        if "vdw" in self.tables:
            self.h_vdw.set_table(self.tables["vdw"][1])
        self.h_atom.set_table(self.tables["elec"][1])
        self.tt_f = self.tables["elec"][1].as_struct()
        return dt

    def step(self, vec: bool = True) -> tuple:
        """One force evaluation (+1/rebuild_every of a list rebuild): returns
        (seconds in reference code, seconds in the CPU restatement)."""
        t_ref = self.t_build[vec] / self.rebuild_every
        t0 = time.perf_counter()
        if self.terms == "lj+ewald":
            self.h_atom.forces("lj", 9.0, vec=vec)
            self.h_atom.forces("ewald_real", 9.0, 0.35, vec=vec)
        if "vdw" in self.terms:
            self.h_vdw.forces("halgren", 9.0, 0.07, 0.12, vec=vec)
        t_ref += time.perf_counter() - t0
        t_port = 0.0
        if "mpole" in self.terms or "polar" in self.terms:
            t0 = time.perf_counter()
            if "mpole" in self.terms:
                self.port.mpole(self.sys, None, 0.5446, 7.0, 332.063713, True, st=self.st,
                                tt=self.tt_f)
            if "polar" in self.terms:
                self.port.perm_field(self.sys, None, 0.5446, 7.0, 0.39, True, st=self.st,
                                     tt=self.tt_f)
            t_port = time.perf_counter() - t0
        if "polar" in self.terms:
            # the reference's own T mat-vec (tmatxb, Thole-only) on the unfiltered
            # list, as many times as the GPU solve applies its operator
            self.h_atom.set_table(self.tables["elec"][0])
            t0 = time.perf_counter()
            for _ in range(self.matvecs):
                self.h_atom.field("tmatxb", 7.0, 0.39, self.mu, vec=vec)
            t_ref += time.perf_counter() - t0
            self.h_atom.set_table(self.tables["elec"][1])
        return t_ref, t_port


def run(config: int, threads: int, repeats: int, warmup: int, seed: int = 1,
        matvecs: int = GPU_PCG_MATVECS, scalar: bool = True, n_mol: int | None = None,
        box: float | None = None) -> dict:
    """`threads` independent replicas (reference shards model), each timed with
    the reference protocol; returns aggregate atom-steps/s (Vec and Scalar)."""
    repeats = max(3, repeats)
    reps = [Replica(config, seed + s, matvecs, n_mol=n_mol, box=box, scalar=scalar)
            for s in range(threads)]
    res = [dict(v=[], s=[], v_port=[]) for _ in range(threads)]

    def work(k):
        r = reps[k]
        for _ in range(warmup):
            if scalar:
                r.step(False)
            r.step(True)
        for _ in range(repeats):
            if scalar:
                a, b = r.step(False)
                res[k]["s"].append(a + b)
            a, b = r.step(True)
            res[k]["v"].append(a + b)
            res[k]["v_port"].append(b)

    th = [threading.Thread(target=work, args=(k,)) for k in range(threads)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    n = reps[0].n
    tv = max(trimmed_mean(r["v"]) for r in res)  # slowest replica
    port = max(trimmed_mean(r["v_port"]) for r in res)
    out = {
        "value": threads * n / tv,
        "unit": "atom-steps/s",
        "cores": threads,
        "s_per_step": tv,
        "port_share": port / tv,
        "wall_s": wall,
        "n_sample_atoms": n,
        "isa": ref_isa(),
        "cpu_model": cpu_model(),
        "repeats": repeats,
        "warmup": warmup,
        "matvecs_per_step": matvecs if "polar" in reps[0].terms else 0,
    }
    if scalar:
        ts = max(trimmed_mean(r["s"]) for r in res)
        out["scalar"] = {"value": threads * n / ts, "s_per_step": ts, "boost": ts / tv}
    return out
