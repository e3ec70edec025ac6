"""Frozen algorithmic FLOP counts per in-cutoff HALF pair.

Weights: add/sub/mul = 1, fma = 2; special functions at their sm_100a
libdevice fast-path cost: div 15, sqrt 13, exp 31, erfc 112; FRND/DSETP are
not flops. Prologue P (3 sub + 3 wrap1 + dist2) = 20. These are the
reference formulation's counts (one evaluation per pair, both sides
updated); the device kernels evaluate each pair once per direction, so the
algorithmic rate they achieve is at most half of their executed rate.
"""

PER_PAIR = {
    "lj": 61 + 12,          # + virial
    "ewald_real": 211 + 12,
    "lj_ewald": 61 + 211 - 20 + 12,  # fused: one prologue
    "halgren": 102 + 12,
    "perm_field_thole": 100,
    "tmatvec_thole": 130,
    "tmatvec": 287,         # Ewald + Thole T
    "tmatvec_pcg": 287,
    "perm_field": 350,      # q + mu + Theta, Ewald + Thole
    "mpole": 570,           # energy + force + torque, q + mu + Theta
}

# neighbour build: algorithmic bytes per rebuild:
# 24 B/atom coordinates read + 4 B per (half) pair written + 8 B/atom offsets.
def nlist_bytes(n_atoms: int, half_pairs: int) -> int:
    return 24 * n_atoms + 4 * half_pairs + 8 * n_atoms
