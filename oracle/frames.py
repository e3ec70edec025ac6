"""ORACLE (test infrastructure only): local multipole frames, SURVEY 8(f)#2.

CPU restatement of paper_1906_01211_b200/csrc/frames.cu in numpy. Frame
types follow Tinker's conventions (the reference has no multipoles, so
parity here is pinned by finite differences of the energy with the frames
rebuilt at displaced positions, tests/test_oracle.py):
  1 z-then-x: z = unit(u), x = unit(v - (v.z) z), y = z x x
  2 bisector: z = unit(unit(u) + unit(v)), x, y as above
u = r_zatom - r_i, v = r_xatom - r_i (minimum image). Global multipoles:
mu = R mu_local, Q = R Q_local R^T with R = [x y z] (columns).

Torque -> force: a frame rotation dtheta changes the energy by -tau.dtheta;
with dz = dtheta x z, dx = dtheta x x the local rotation components are
dth_x = -y.dz, dth_y = x.dz, dth_z = y.dx, hence
dE/du = -(-tau_x Jzu^T y + tau_y Jzu^T x + tau_z Jxu^T y) (and for v), with
the Jacobians written here by differentiating the axis formulas.
"""
from __future__ import annotations

import numpy as np


def _wrap(d, box):
    box = np.asarray(box, float)
    return d - box * np.rint(d / box)


def _unit_jac(w):
    """unit(w) and its Jacobian (I - e e^T)/|w|."""
    lw = np.linalg.norm(w)
    e = w / lw
    return e, (np.eye(3) - np.outer(e, e)) / lw


def frame_axes(kind: int, u, v, jac: bool = False):
    u = np.asarray(u, float)
    v = np.asarray(v, float)
    if kind == 2:
        uh, ju = _unit_jac(u)
        vh, jv = _unit_jac(v)
        z, jz = _unit_jac(uh + vh)
        jzu, jzv = jz @ ju, jz @ jv
    elif kind == 1:
        z, jzu = _unit_jac(u)
        jzv = np.zeros((3, 3))
    else:
        raise ValueError("frame type must be 1 or 2")
    vz = v @ z
    w = v - vz * z
    x, jx = _unit_jac(w)
    y = np.cross(z, x)
    if not jac:
        return x, y, z
    a = np.outer(z, v) + vz * np.eye(3)       # d(z (z.v))/dz
    dwu = -(a @ jzu)
    dwv = np.eye(3) - np.outer(z, z) - a @ jzv
    return x, y, z, jzu, jzv, jx @ dwu, jx @ dwv


def rotate(pos, box, frame, zatom, xatom, dip_local, quad_local):
    """Global (dipole (n,3), quadrupole (n,6)) from the local ones."""
    n = len(frame)
    dip = np.array(dip_local, float).reshape(n, 3).copy()
    quad = np.array(quad_local, float).reshape(n, 6).copy()
    for i in range(n):
        if frame[i] == 0:
            continue
        u = _wrap(pos[zatom[i]] - pos[i], box)
        v = _wrap(pos[xatom[i]] - pos[i], box)
        x, y, z = frame_axes(int(frame[i]), u, v)
        R = np.stack([x, y, z], 1)
        q = quad_local[i]
        Q = np.array([[q[0], q[1], q[2]], [q[1], q[3], q[4]], [q[2], q[4], q[5]]])
        G = R @ Q @ R.T
        dip[i] = R @ np.asarray(dip_local[i], float)
        quad[i] = [G[0, 0], G[0, 1], G[0, 2], G[1, 1], G[1, 2], G[2, 2]]
    return dip, quad


def torque_forces(pos, box, frame, zatom, xatom, torque):
    """Forces (n, 3) on the frame atoms equivalent to the site torques."""
    n = len(frame)
    f = np.zeros((n, 3))
    for i in range(n):
        if frame[i] == 0:
            continue
        u = _wrap(pos[zatom[i]] - pos[i], box)
        v = _wrap(pos[xatom[i]] - pos[i], box)
        x, y, z, jzu, jzv, jxu, jxv = frame_axes(int(frame[i]), u, v, jac=True)
        t = np.asarray(torque[i], float)
        tx, ty, tz = t @ x, t @ y, t @ z
        gu = -(-tx * jzu.T @ y + ty * jzu.T @ x + tz * jxu.T @ y)
        gv = -(-tx * jzv.T @ y + ty * jzv.T @ x + tz * jxv.T @ y)
        f[zatom[i]] -= gu
        f[xatom[i]] -= gv
        f[i] += gu + gv
    return f


def water_frames(molecule):
    """Tinker water frames for molecules of (O, H, H): O bisector of the two
    H, each H z-then-x (z toward O, x toward the other H)."""
    mol = np.asarray(molecule)
    n = len(mol)
    frame = np.zeros(n, np.int32)
    za = np.zeros(n, np.int32)
    xa = np.zeros(n, np.int32)
    for o in range(0, n, 3):
        h1, h2 = o + 1, o + 2
        frame[o], za[o], xa[o] = 2, h1, h2
        frame[h1], za[h1], xa[h1] = 1, o, h2
        frame[h2], za[h2], xa[h2] = 1, o, h1
    return frame, za, xa
