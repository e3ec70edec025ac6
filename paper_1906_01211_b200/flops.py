"""Frozen algorithmic work per unit for the roofline.

FP64-bound kernels: FLOPs per in-cutoff HALF pair. Weights: add/sub/mul = 1,
fma = 2; special functions at their sm_100a libdevice fast-path cost: div 15,
sqrt 13, exp 31, erfc 112; FRND/DSETP are not flops. Prologue P (3 sub +
3 wrap1 + dist2) = 20. These are the reference formulation's counts (one
evaluation per pair, both sides updated). The default device kernels do the
same (half rows, partner update by atomics); field_tpre and the deterministic
mode evaluate each pair once per direction, so there the algorithmic rate is
at most half of the executed rate.

HBM-bound kernels: algorithmic DRAM bytes per launch (streamed list slots
plus per-site vectors; gathers of neighbour data are cache traffic).
"""

PER_PAIR_FLOPS = {
    "lj": 61 + 12,          # + virial
    "ewald_real": 211 + 12,
    "lj_ewald": 61 + 211 - 20 + 12,  # fused: one prologue
    "halgren": 102 + 12,
    "perm_field_thole": 100,
    "tmatvec_thole": 130,
    "tmatvec": 287,         # Ewald + Thole T, recomputed per call
    "perm_field": 350,      # q + mu + Theta, Ewald + Thole
    "field_tpre": 350,      # the same field; the T tensors it stores are a by-product
    "mpole": 570,           # energy + force + torque, q + mu + Theta
    # polarization forces (8(f)#1): P + Thole l3..l9 (exp + 12) + Ewald B0..4
    # (erfc + exp + sqrt + div + 16) + rr3..9 (12) + h (25) + f, g with
    # gradients (2 x 75) + dipole/quadrupole torques on both sites (2 x 60)
    "polar_force": 20 + 43 + 187 + 12 + 25 + 150 + 120,
}

# (kernel) -> which pairs its unit counts: (list role, cutoff key, excluded?)
PAIRS_OF = {
    "lj": ("elec", "cutoff", True), "ewald_real": ("elec", "cutoff", True),
    "lj_ewald": ("elec", "cutoff", True), "halgren": ("vdw", "vdw_cutoff", True),
    "mpole": ("elec", "elec_cutoff", True), "perm_field": ("elec", "elec_cutoff", True),
    "field_tpre": ("elec", "elec_cutoff", True), "tmatvec": ("elec", "elec_cutoff", False),
    "tmatvec_pcg": ("elec", "elec_cutoff", False), "tmatvec_pre": ("elec", "elec_cutoff", False),
    "polar_force": ("elec", "elec_cutoff", False),
}


def stream_bytes(kernel: str, n_atoms: int, directed_pairs: int) -> int | None:
    """Algorithmic DRAM bytes of one launch of an HBM-bound kernel."""
    if kernel in ("tmatvec_pcg", "tmatvec_pre"):
        # per directed pair: 4 B index + 16 B (rr3, rr5); per site: count,
        # position, p, alpha (read) + q (write)
        return 20 * directed_pairs + (4 + 32 + 32 + 16 + 32) * n_atoms
    if kernel == "prune":
        return 4 * directed_pairs * 2 + 4 * n_atoms  # read 9 A slots ~2x, write 7 A slots
    return None


def nlist_bytes(n_atoms: int, half_pairs: int) -> int:
    """Neighbour build, per rebuild: 24 B/atom coordinates read + 4 B per
    (half) pair written + 8 B/atom offsets."""
    return 24 * n_atoms + 4 * half_pairs + 8 * n_atoms
