"""ORACLE (test infrastructure only): reciprocal-space Ewald for point
charges by the direct structure-factor sum, SURVEY 8(f)#3.

The reference has no reciprocal space (real space only); this is
the textbook Ewald sum, exact up to the k-space cutoff (converged here to
double precision for the small systems the tests use), against which the
device's smooth-PME (B-splines + FFT) is checked at PME accuracy. With R =
the real-space part (proj/include/mdvec/kernels.hpp:57-68 times electric),
the total R + recip + self + excluded-pair correction is independent of
alpha -- a second, oracle-free check.

  E_recip = 1/(2 pi V) sum_{m != 0} exp(-pi^2 m^2 / a^2) / m^2 |S(m)|^2
  S(m)    = sum_j q_j exp(2 pi i m.r_j),  m = (k1/Lx, k2/Ly, k3/Lz)
  F_i     = (2 q_i / V) sum_m exp(-pi^2 m^2/a^2)/m^2 m Im[exp(2 pi i m.r_i) conj(S)]
  E_self  = -a/sqrt(pi) sum q^2
  E_excl  = -sum_{excluded pairs} q_i q_j erf(a r)/r   (the reciprocal sum
            contains the excluded pairs; this removes them)
All energies times `electric`.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf


def recip(pos, q, box, alpha, kmax=(12, 12, 12), electric=1.0):
    """(energy, forces (n,3), virial 3x3) of the reciprocal sum."""
    box = np.asarray(box, float)
    V = float(np.prod(box))
    k = [np.arange(-km, km + 1) for km in kmax]
    K1, K2, K3 = np.meshgrid(*k, indexing="ij")
    m = np.stack([K1.ravel() / box[0], K2.ravel() / box[1], K3.ravel() / box[2]], 1)
    m2 = np.sum(m * m, 1)
    keep = m2 > 0
    m, m2 = m[keep], m2[keep]
    g = np.exp(-np.pi ** 2 * m2 / alpha ** 2) / m2          # (M,)
    phase = 2.0 * np.pi * (np.asarray(pos) @ m.T)            # (n, M)
    c, s = np.cos(phase), np.sin(phase)
    Sr = q @ c
    Si = q @ s
    S2 = Sr ** 2 + Si ** 2
    e = electric * np.sum(g * S2) / (2.0 * np.pi * V)
    # Im[exp(i phi_i) conj(S)] = sin(phi_i) Sr - cos(phi_i) Si
    im = s * Sr[None, :] - c * Si[None, :]
    f = electric * (2.0 / V) * q[:, None] * ((im * g[None, :]) @ m)
    # virial W_ab = sum_k E_k (delta_ab - 2 (1 + pi^2 m^2/a^2) m_a m_b / m^2)
    ek = electric * g * S2 / (2.0 * np.pi * V)
    fac = 2.0 * (1.0 + np.pi ** 2 * m2 / alpha ** 2) / m2
    w = np.eye(3) * np.sum(ek) - np.einsum("k,ka,kb->ab", ek * fac, m, m)
    return e, f, w


def self_energy(q, alpha, electric=1.0):
    return -electric * alpha / np.sqrt(np.pi) * float(np.sum(np.asarray(q) ** 2))


def excluded_correction(pos, q, box, molecule, alpha, electric=1.0):
    """(energy, forces, virial) removing the excluded (same-molecule) pairs
    from the reciprocal sum: -q_i q_j erf(a r)/r per pair."""
    pos = np.asarray(pos, float)
    box = np.asarray(box, float)
    n = len(q)
    f = np.zeros((n, 3))
    w = np.zeros((3, 3))
    e = 0.0
    mol = np.asarray(molecule)
    for i in range(n):
        for j in range(i + 1, n):
            if mol[i] != mol[j]:
                continue
            d = pos[i] - pos[j]
            d -= box * np.rint(d / box)
            r = np.sqrt(d @ d)
            qq = electric * q[i] * q[j]
            e -= qq * erf(alpha * r) / r
            # d/dr [erf(a r)/r] = (2a/sqrt(pi) exp(-a^2 r^2) - erf(a r)/r) / r
            dd = (2 * alpha / np.sqrt(np.pi) * np.exp(-alpha ** 2 * r * r) - erf(alpha * r) / r) / r
            fi = qq * dd * d / r  # F_i = -dE/dr_i = +qq d/dr(erf/r) * rhat
            f[i] += fi
            f[j] -= fi
            w += np.outer(d, fi)
    return e, f, w
