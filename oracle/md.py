"""ORACLE (test infrastructure only): harmonic bonded terms and a velocity
Verlet integrator in numpy, SURVEY 8(f)#4 -- the restatement of
paper_1906_01211_b200/csrc/md.cu the device trajectory is compared with.

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
