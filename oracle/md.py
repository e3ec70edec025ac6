"""ORACLE (test infrastructure only): harmonic bonded terms, a velocity
Verlet integrator and the two-level BAOAB-RESPA Langevin integrator in numpy,
SURVEY 8(f)#4 -- the restatement of paper_1906_01211_b200/csrc/md.cu (and
mdg_md_run in csrc/abi.cpp) the device trajectory is compared with. The
multi-timestep Langevin scheme is the one /root/reference/PAPER.md:782-783
names for the paper's Rel2 (BAOAB splitting; RESPA levels: bonded inside,
nonbonded outside).

Units kcal/mol, A, amu, fs; a = F/m * 4.184e-4. Bond energy kb (r - r0)^2,
angle energy ka (theta - theta0)^2 (theta in radians, vertex in the middle).
"""
from __future__ import annotations

import numpy as np

ACCEL = 4.184e-4


def _wrap(d, box):
    return d - box * np.rint(d / box)


def bonded(pos, box, bonds, kb, r0, angles, ka, th0):
    """(energy_bonds, energy_angles, forces (n, 3))."""
    box = np.asarray(box, float)
    f = np.zeros_like(pos)
    eb = ea = 0.0
    for (i, j), k, r0_ in zip(bonds, np.broadcast_to(kb, len(bonds)),
                              np.broadcast_to(r0, len(bonds))):
        d = _wrap(pos[i] - pos[j], box)
        r = np.sqrt(d @ d)
        eb += k * (r - r0_) ** 2
        g = -2.0 * k * (r - r0_) / r * d
        f[i] += g
        f[j] -= g
    for (i, j, k_), k, t0 in zip(angles, np.broadcast_to(ka, len(angles)),
                                 np.broadcast_to(th0, len(angles))):
        a = _wrap(pos[i] - pos[j], box)
        c = _wrap(pos[k_] - pos[j], box)
        ra, rc = np.sqrt(a @ a), np.sqrt(c @ c)
        cs = np.clip(a @ c / (ra * rc), -1.0, 1.0)
        th = np.arccos(cs)
        ea += k * (th - t0) ** 2
        sn = max(np.sqrt(max(0.0, 1 - cs * cs)), 1e-12)
        de = 2.0 * k * (th - t0)
        fi = de / (sn * ra) * (c / rc - cs * a / ra)
        fk = de / (sn * rc) * (a / ra - cs * c / rc)
        f[i] += fi
        f[k_] += fk
        f[j] -= fi + fk
    return eb, ea, f


def kinetic(vel, mass):
    return 0.5 * float(np.sum(np.asarray(mass)[:, None] * vel * vel)) / ACCEL


def velocity_verlet(pos, vel, mass, box, force_fn, dt, nsteps):
    """force_fn(pos) -> (forces, potential); positions wrapped into [0, L).
    Returns final (pos, vel) and per-step (kinetic, potential)."""
    box = np.asarray(box, float)
    inv = ACCEL / np.asarray(mass, float)[:, None]
    pos = np.array(pos, float)
    vel = np.array(vel, float)
    f, _ = force_fn(pos)
    ek, ep = [], []
    for _ in range(nsteps):
        vel += 0.5 * dt * inv * f
        pos = pos + dt * vel
        pos -= box * np.floor(pos / box)
        f, u = force_fn(pos)
        vel += 0.5 * dt * inv * f
        ek.append(kinetic(vel, mass))
        ep.append(u)
    return pos, vel, np.array(ek), np.array(ep)


def water_topology(n_mol: int):
    """O-H bonds and the H-O-H angle of n_mol (O, H, H) waters."""
    bonds, angles = [], []
    for m in range(n_mol):
        o = 3 * m
        bonds += [(o, o + 1), (o, o + 2)]
        angles.append((o + 1, o, o + 2))
    return np.array(bonds, np.int32), np.array(angles, np.int32)


KB = 0.0019872041  # kcal/mol/K


def splitmix64(x):
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic), as
    md.cu splitmix64."""
    x = np.asarray(x, np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def gauss(seed: int, counter: int, n: int):
    """(n, 3) normal deviates of md.cu k_ostep for caller sites 0..n-1."""
    with np.errstate(over="ignore"):
        s0 = splitmix64(np.array([counter], np.uint64))
        base = splitmix64(np.array([seed], np.uint64) + s0)
        key = base + np.uint64(3) * np.arange(n, dtype=np.uint64)[:, None] \
            + np.arange(3, dtype=np.uint64)[None, :]
        h = splitmix64(key)
    u1 = ((h >> np.uint64(32)) + np.uint64(1)).astype(np.float64) * 2.0 ** -32
    u2 = (h & np.uint64(0xFFFFFFFF)).astype(np.float64) * 2.0 ** -32
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def baoab_respa(pos, vel, mass, box, slow_fn, fast_fn, dt, n_inner, friction_ps,
                temperature_k, seed, nsteps):
    """Two-level BAOAB-RESPA (md.cu / abi.cpp mdg_md_run):
    B_out(dt/2) [B_in(h/2) A(h/2) O(h) A(h/2) F_in B_in(h/2)] x n_inner F_out
    B_out(dt/2), h = dt / n_inner, O: v = c1 v + sqrt((1 - c1^2) kT/m) xi.
    slow_fn / fast_fn(pos) -> (forces, potential). Returns final (pos, vel)
    and per-step (kinetic, slow + fast potential)."""
    box = np.asarray(box, float)
    m = np.asarray(mass, float)
    inv = ACCEL / m[:, None]
    pos = np.array(pos, float)
    vel = np.array(vel, float)
    h = dt / n_inner
    c1 = np.exp(-friction_ps * 1e-3 * h)
    c2 = np.sqrt(max(0.0, 1.0 - c1 * c1))
    sig = c2 * np.sqrt(KB * temperature_k * ACCEL * (1.0 / m))[:, None]
    fs, us = slow_fn(pos)
    ff, uf = fast_fn(pos)
    counter = 0
    ek, ep = [], []

    def drift(p, t):
        p = p + t * vel
        return p - box * np.floor(p / box)

    for _ in range(nsteps):
        vel += 0.5 * dt * inv * fs
        for _k in range(n_inner):
            vel += 0.5 * h * inv * ff
            pos = drift(pos, 0.5 * h)
            if friction_ps > 0:
                vel = c1 * vel + sig * gauss(seed, counter, len(m))
                counter += 1
            pos = drift(pos, 0.5 * h)
            ff, uf = fast_fn(pos)
            vel += 0.5 * h * inv * ff
        fs, us = slow_fn(pos)
        vel += 0.5 * dt * inv * fs
        ek.append(kinetic(vel, mass))
        ep.append(us + uf)
    return pos, vel, np.array(ek), np.array(ep)
