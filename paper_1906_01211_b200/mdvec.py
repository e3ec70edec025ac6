"""Python mirror of the reference `mdvec` API over the C ABI (include/mdg.h).

Same names, argument meaning and error behaviour as the reference's C++
headers (proj/include/mdvec/{neighbors,kernels,polar}.hpp): kernels take a
system, a neighbour table and a params struct and OVERWRITE their output;
failures raise ContractViolation / CapacityError / SingularityError /
ConvergenceError (proj/include/mdvec/common.hpp:12-32). Every call runs on
the GPU through libmdg.so; there is no CPU fallback -- if the library or a
device is missing, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MDG_LIB points at an alternative build of the same ABI (kernel experiments)
LIB_PATH = os.environ.get("MDG_LIB", os.path.join(_HERE, "libmdg.so"))
ROOT = os.path.dirname(_HERE)

def _aos(x, y, z):
    """(n, 3) view of three SoA component arrays: no copy when they are
    consecutive rows of one (3, n) block (as Engine._vec3 and host_array
    blocks are), else a stacked copy."""
    n = len(x)
    step = n * x.itemsize
    if (n and x.dtype == y.dtype == z.dtype and x.flags.c_contiguous and y.flags.c_contiguous
            and z.flags.c_contiguous and y.ctypes.data - x.ctypes.data == step
            and z.ctypes.data - y.ctypes.data == step):
        return np.lib.stride_tricks.as_strided(x, shape=(n, 3), strides=(x.itemsize, step),
                                               writeable=True)
    return np.stack([x, y, z], 1)


kMaxNeighbors = 2560  # proj/include/mdvec/common.hpp:10
SITES_ATOMIC, SITES_VDW = 0, 1
ELECTRIC = 332.063713  # kcal A / (mol e^2)
DEBYE = 4.80321        # D per e A


# ---- error taxonomy (proj/include/mdvec/common.hpp:12-32) --------------------
class MdgError(RuntimeError):
    code = -1


class ContractViolation(MdgError, ValueError):
    code = 1


class CapacityError(MdgError):
    code = 2


class SingularityError(MdgError, ArithmeticError):
    code = 3


class ConvergenceError(MdgError):
    code = 4

    def __init__(self, msg, last_residual=float("nan")):
        super().__init__(msg)
        self.last_residual = last_residual


class CudaError(MdgError):
    code = 5


class CommError(MdgError):
    code = 6


_ERRORS = {1: ContractViolation, 2: CapacityError, 3: SingularityError, 4: ConvergenceError,
           5: CudaError, 6: CommError}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint32)
_lp = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)

# every exported symbol of include/mdg.h with its ctypes signature
SIGNATURES = {
    "mdg_last_error": (C.c_char_p, []),
    "mdg_version": (C.c_int, []),
    "mdg_ctx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_int32]),
    "mdg_ctx_destroy": (C.c_int, [C.c_void_p]),
    "mdg_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "mdg_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "mdg_system_upload": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_double]
                          + [_dp] * 9),
    "mdg_positions_upload": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_topology_upload": (C.c_int, [C.c_void_p, _ip, _ip, _dp]),
    "mdg_multipoles_upload": (C.c_int, [C.c_void_p, _dp, _dp]),
    "mdg_nlist_build": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int]),
    "mdg_nlist_size": (C.c_int, [C.c_void_p, C.c_int, _i64p, _i64p]),
    "mdg_nlist_export": (C.c_int, [C.c_void_p, C.c_int, _up, _up, _up, _lp, _ip, C.c_int64]),
    "mdg_nlist_import": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int, _up, _lp, _ip]),
    "mdg_lj_forces": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp,
                                _dp, _dp, _dp]),
    "mdg_ewald_real_forces": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_int, _dp, _dp, _dp, _dp, _dp]),
    "mdg_halgren_forces": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_int, _dp, _dp, _dp, _dp, _dp]),
    "mdg_tmatvec": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp,
                              _dp, _dp, _dp, _dp]),
    "mdg_perm_field": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.c_int, _dp, _dp, _dp]),
    "mdg_polar_solve_jacobi": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                         C.c_double, C.c_int64, _dp, _dp, _dp, _i64p, _dp]),
    "mdg_polar_solve_pcg": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_int, C.c_double, C.c_int64, _dp, _dp, _dp, _i64p,
                                      _dp]),
    "mdg_mpole_forces": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "mdg_polar_forces": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                   _dp, _dp, _dp, _dp]),
    "mdg_ewald_recip": (C.c_int, [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp]),
    "mdg_ewald_recip_mpole": (C.c_int, [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                        _dp, _dp]),
    "mdg_set_ewald_recip": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    "mdg_resort": (C.c_int, [C.c_void_p]),
    "mdg_charmm_step": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "mdg_bonded_upload": (C.c_int, [C.c_void_p, C.c_int64, _ip, _dp, _dp, C.c_int64, _ip, _dp,
                                    _dp]),
    "mdg_bonded_forces": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp]),
    "mdg_velocities_upload": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp]),
    "mdg_velocities_fetch": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_positions_fetch": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_md_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _dp, _dp]),
    "mdg_amoeba_step": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "mdg_fetch_forces": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_fetch_torques": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_fetch_dipoles": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_fetch_energies": (C.c_int, [C.c_void_p, _dp, _dp, _i64p, _dp]),
    "mdg_fetch_perm_field": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_launch_count": (C.c_int64, [C.c_void_p]),
    "mdg_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_profile_reset": (C.c_int, [C.c_void_p]),
    "mdg_profile_report": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "mdg_system_upload_owned": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                          C.c_double, C.c_double, C.c_double] + [_dp] * 9),
    "mdg_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "mdg_group_create_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int,
                                         C.POINTER(C.c_void_p), C.c_int64]),
    "mdg_group_create_nccl": (C.c_int, [C.POINTER(C.c_void_p), C.c_void_p, C.c_int, C.c_int,
                                        C.c_void_p, C.c_int64]),
    "mdg_group_destroy": (C.c_int, [C.c_void_p]),
    "mdg_md_rebuild_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "mdg_positions_upload_owned": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_group_set_overlap": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_group_set_halo_local": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, _ip, _ip, _ip]),
    "mdg_group_set_halo_nccl": (C.c_int, [C.c_void_p, C.c_int, _ip, _i64p, _ip, _i64p, _ip]),
    "mdg_group_exchange": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_group_allreduce_results": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "mdg_group_set_reference": (C.c_int, [C.c_void_p]),
    "mdg_group_max_displacement": (C.c_int, [C.c_void_p, _dp]),
    "mdg_group_amoeba_step": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "mdg_group_charmm_step": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "mdg_group_fetch_energies": (C.c_int, [C.c_void_p, _dp, _dp, _i64p, _dp]),
    "mdg_set_deterministic": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_set_debug_perturb": (C.c_int, [C.c_void_p, C.c_double]),
    "mdg_frames_upload": (C.c_int, [C.c_void_p, _ip, _ip, _ip, _dp, _dp]),
    "mdg_set_overlap": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_set_cluster_matvec": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_set_cluster_halgren": (C.c_int, [C.c_void_p, C.c_int]),
    "mdg_vec_pack": (C.c_int, [C.c_void_p, C.c_int, _ip, C.c_int64, _dp]),
    "mdg_vec_unpack": (C.c_int, [C.c_void_p, C.c_int, _ip, C.c_int64, _dp]),
    "mdg_vec_pack_dev": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]),
    "mdg_vec_unpack_dev": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]),
    "mdg_timer_start": (C.c_int, [C.c_void_p]),
    "mdg_timer_stop": (C.c_int, [C.c_void_p, _dp]),
    "mdg_probe_fp64_peak": (C.c_int, [C.c_int, _dp]),
    "mdg_probe_erfc": (C.c_int, [C.c_int, _dp, C.c_int64, _dp]),
    "mdg_host_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_int64]),
    "mdg_host_free": (C.c_int, [C.c_void_p]),
    "mdg_set_force_output": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "mdg_nlist_count_within": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int, _i64p,
                                         _i64p]),
    "mdg_water_generate": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, C.c_int, _dp, _dp, _dp,
                                     _ip, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _dp, _dp, _dp]),
    "mdg_reduce_sites_host": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_double, _dp, _dp,
                                        _dp, _ip, _dp, _dp, _dp, _dp]),
}


class CharmmParams(C.Structure):
    _fields_ = [("cutoff", C.c_double), ("alpha", C.c_double), ("electric", C.c_double),
                ("shift", C.c_int), ("exclude", C.c_int)]


class AmoebaParams(C.Structure):
    _fields_ = [("vdw_cutoff", C.c_double), ("delta", C.c_double), ("gamma", C.c_double),
                ("elec_cutoff", C.c_double), ("alpha", C.c_double), ("electric", C.c_double),
                ("thole_a", C.c_double), ("tol_debye", C.c_double), ("max_iter", C.c_int64),
                ("exclude", C.c_int), ("terms", C.c_int)]


TERM_VDW, TERM_MPOLE, TERM_POLAR, TERM_POLAR_FORCE = 1, 2, 4, 8


INTEGRATOR_VERLET = 0
INTEGRATOR_BAOAB_RESPA = 1
PREDICT_NONE = 0
PREDICT_ASPC = 1


class MDParams(C.Structure):
    """mdg.h mdg_md_params."""
    _fields_ = [("model", C.c_int), ("nsteps", C.c_int64), ("dt_fs", C.c_double),
                ("rebuild_every", C.c_int), ("elec_list", C.c_int), ("vdw_list", C.c_int),
                ("elec_list_cutoff", C.c_double), ("vdw_list_cutoff", C.c_double),
                ("bonded", C.c_int),
                # zero defaults keep velocity Verlet
                ("integrator", C.c_int), ("inner_steps", C.c_int),
                ("friction_ps", C.c_double), ("temperature_k", C.c_double),
                ("seed", C.c_uint64), ("predictor", C.c_int)]


_lib = None


def load_library(path: str | None = None):
    """Load libmdg.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} is missing: build it with `make -C {_HERE}` "
                          "(the product has no CPU fallback)")
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def check(rc: int, extra: float | None = None):
    if rc == 0:
        return
    msg = load_library().mdg_last_error().decode()
    cls = _ERRORS.get(rc, MdgError)
    if cls is ConvergenceError:
        raise ConvergenceError(msg, extra if extra is not None else float("nan"))
    raise cls(msg)


# ---- reference data types --------------------------------------------------------
@dataclass
class ParticleSystem:
    """proj/include/mdvec/system.hpp:12-25 plus the topology/multipole extensions."""
    box: tuple
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    charge: np.ndarray
    lj_sigma: np.ndarray
    lj_epsilon: np.ndarray
    hal_r0: np.ndarray
    hal_epsilon: np.ndarray
    polarizability: np.ndarray
    molecule: np.ndarray | None = None
    dipole: np.ndarray | None = None
    quadrupole: np.ndarray | None = None
    hred_parent: np.ndarray | None = None
    hred_factor: np.ndarray | None = None

    @property
    def n_sites(self) -> int:
        return int(len(self.x))


@dataclass
class LjParams:  # proj/include/mdvec/kernels.hpp:11-14
    cutoff: float
    shift: bool = False


@dataclass
class EwaldRealParams:  # proj/include/mdvec/kernels.hpp:16-19
    alpha: float
    cutoff: float


@dataclass
class HalgrenParams:  # proj/include/mdvec/polar.hpp:8-12
    cutoff: float
    delta: float = 0.07
    gamma: float = 0.12


@dataclass
class PolarParams:  # proj/include/mdvec/polar.hpp:14-17
    cutoff: float
    thole_a: float = 0.39


@dataclass
class ForceAccumulator:  # proj/include/mdvec/kernels.hpp:21-34 (+ virial)
    fx: np.ndarray
    fy: np.ndarray
    fz: np.ndarray
    energy: float = 0.0
    virial: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))

    @property
    def forces(self) -> np.ndarray:
        return np.stack([self.fx, self.fy, self.fz], 1)


@dataclass
class FieldArrays:  # proj/include/mdvec/polar.hpp:74-84
    ex: np.ndarray
    ey: np.ndarray
    ez: np.ndarray

    @property
    def field(self) -> np.ndarray:
        return np.stack([self.ex, self.ey, self.ez], 1)


@dataclass
class PolarizationState:  # proj/include/mdvec/system.hpp:36-42
    mu_x: np.ndarray
    mu_y: np.ndarray
    mu_z: np.ndarray
    thole_a: float = 0.39
    iterations: int = 0
    last_residual: float = 0.0

    @property
    def mu(self) -> np.ndarray:
        return np.stack([self.mu_x, self.mu_y, self.mu_z], 1)


@dataclass
class NeighborTable:
    """Handle to a device list plus the reference layout on demand
    (proj/include/mdvec/neighbors.hpp:22-41)."""
    engine: "Engine"
    list_id: int
    cutoff: float
    sites: int

    @property
    def n_sites(self) -> int:
        return self.engine.n

    def export(self):
        return self.engine.export_table(self)

    def pairs(self) -> np.ndarray:
        """table_pairs(): canonical sorted (i<j) pairs (proj/src/neighbors.cpp:59-72)."""
        nn, _, _, off, idx = self.export()
        rows = [np.stack([np.full(nn[i], i, np.int64), idx[off[i]: off[i] + nn[i]]], 1)
                for i in range(len(nn))]
        p = np.concatenate(rows) if rows else np.zeros((0, 2), np.int64)
        o = np.lexsort((p[:, 1], p[:, 0]))
        return p[o]


class Engine:
    """One device context (mdg_ctx): a GPU, a stream, preallocated capacity."""

    def __init__(self, n_capacity: int, device: int = 0, max_pairs_per_atom: int = 0):
        self.lib = load_library()
        self.ctx = C.c_void_p()
        check(self.lib.mdg_ctx_create(C.byref(self.ctx), device, int(n_capacity),
                                      int(max_pairs_per_atom)))
        self.n = 0
        self.box = None
        self._next_list = 0

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            self.lib.mdg_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- uploads ---------------------------------------------------------------
    def upload_system(self, s) -> None:
        """mdg_system_upload + topology + multipoles from a ParticleSystem-like object."""
        arrs = [_f64(getattr(s, k)) for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon",
                                               "hal_r0", "hal_epsilon", "polarizability")]
        self._keep = arrs
        check(self.lib.mdg_system_upload(self.ctx, len(arrs[0]), *map(float, s.box),
                                         *(_p(a) for a in arrs)))
        self.n = len(arrs[0])
        self.box = tuple(map(float, s.box))
        mol = getattr(s, "molecule", None)
        par = getattr(s, "hred_parent", None)
        fac = getattr(s, "hred_factor", None)
        if mol is not None or par is not None:
            self.upload_topology(mol, par, fac)
        dip = getattr(s, "dipole", None)
        quad = getattr(s, "quadrupole", None)
        if dip is not None or quad is not None:
            self.upload_multipoles(dip, quad)

    def vec_pack(self, vec_id: int, sites) -> np.ndarray:
        """3 doubles per listed (caller-order) site of a device vector."""
        idx = np.ascontiguousarray(sites, np.int32)
        out = np.zeros(3 * len(idx))
        check(self.lib.mdg_vec_pack(self.ctx, vec_id, _p(idx, _ip), len(idx), _p(out)))
        return out

    def vec_unpack(self, vec_id: int, sites, data) -> None:
        idx = np.ascontiguousarray(sites, np.int32)
        buf = _f64(data)
        check(self.lib.mdg_vec_unpack(self.ctx, vec_id, _p(idx, _ip), len(idx), _p(buf)))

    def upload_positions(self, x, y, z):
        x, y, z = _f64(x), _f64(y), _f64(z)
        check(self.lib.mdg_positions_upload(self.ctx, _p(x), _p(y), _p(z)))

    def upload_positions_owned(self, x, y, z):
        """A domain context's owned coordinates (mdg_positions_upload_owned);
        page-locked arrays (host_array) are DMA'd without a staging copy."""
        x, y, z = _f64(x), _f64(y), _f64(z)
        check(self.lib.mdg_positions_upload_owned(self.ctx, _p(x), _p(y), _p(z)))

    def upload_topology(self, molecule=None, hred_parent=None, hred_factor=None):
        m = None if molecule is None else np.ascontiguousarray(molecule, np.int32)
        p = None if hred_parent is None else np.ascontiguousarray(hred_parent, np.int32)
        f = None if hred_factor is None else _f64(hred_factor)
        check(self.lib.mdg_topology_upload(self.ctx, _p(m, _ip), _p(p, _ip), _p(f)))

    def upload_multipoles(self, dipole=None, quadrupole=None):
        d = None if dipole is None else _f64(np.asarray(dipole).reshape(-1))
        q = None if quadrupole is None else _f64(np.asarray(quadrupole).reshape(-1))
        check(self.lib.mdg_multipoles_upload(self.ctx, _p(d), _p(q)))

    # ---- lists -------------------------------------------------------------------
    def build_neighbor_table(self, list_cutoff: float, list_id: int | None = None,
                             sites: int = SITES_ATOMIC) -> NeighborTable:
        """build_cell_grid + build_neighbor_table (proj/include/mdvec/neighbors.hpp:43-50)."""
        if list_id is None:
            list_id = 0 if sites == SITES_ATOMIC else 1
        check(self.lib.mdg_nlist_build(self.ctx, list_id, float(list_cutoff), sites))
        return NeighborTable(self, list_id, float(list_cutoff), sites)

    def import_table(self, nnvlst, offset, indices, cutoff: float, list_id: int = 2,
                     sites: int = SITES_ATOMIC) -> NeighborTable:
        nn = np.ascontiguousarray(nnvlst, np.uint32)
        off = np.ascontiguousarray(offset, np.uint64)
        idx = np.ascontiguousarray(indices, np.int32)
        check(self.lib.mdg_nlist_import(self.ctx, list_id, float(cutoff), sites, _p(nn, _up),
                                        _p(off, _lp), _p(idx, _ip)))
        return NeighborTable(self, list_id, float(cutoff), sites)

    def table_size(self, t: NeighborTable):
        hp, ps = C.c_int64(), C.c_int64()
        check(self.lib.mdg_nlist_size(self.ctx, t.list_id, C.byref(hp), C.byref(ps)))
        return hp.value, ps.value

    def export_table(self, t: NeighborTable):
        _, total = self.table_size(t)
        n = self.n
        nn, n8, n16 = (np.zeros(n, np.uint32) for _ in range(3))
        off = np.zeros(n, np.uint64)
        idx = np.zeros(max(total, 1), np.int32)
        check(self.lib.mdg_nlist_export(self.ctx, t.list_id, _p(nn, _up), _p(n8, _up),
                                        _p(n16, _up), _p(off, _lp), _p(idx, _ip), len(idx)))
        return nn, n8, n16, off, idx[:total]

    # ---- kernels -------------------------------------------------------------------
    def _vec3(self):
        # three rows of one (3, n) block: _aos() returns its (n, 3) view
        # without another copy of the data
        b = np.zeros((3, self.n))
        return b[0], b[1], b[2]

    def lj_forces(self, t: NeighborTable, p: LjParams, exclude: bool = False) -> ForceAccumulator:
        fx, fy, fz = self._vec3()
        e = C.c_double()
        w = np.zeros(9)
        check(self.lib.mdg_lj_forces(self.ctx, t.list_id, p.cutoff, int(p.shift), int(exclude),
                                     _p(fx), _p(fy), _p(fz), C.byref(e), _p(w)))
        return ForceAccumulator(fx, fy, fz, e.value, w.reshape(3, 3))

    def ewald_real_forces(self, t: NeighborTable, p: EwaldRealParams, electric: float = 1.0,
                          exclude: bool = False) -> ForceAccumulator:
        fx, fy, fz = self._vec3()
        e = C.c_double()
        w = np.zeros(9)
        check(self.lib.mdg_ewald_real_forces(self.ctx, t.list_id, p.alpha, p.cutoff, electric,
                                             int(exclude), _p(fx), _p(fy), _p(fz), C.byref(e),
                                             _p(w)))
        return ForceAccumulator(fx, fy, fz, e.value, w.reshape(3, 3))

    def halgren_forces(self, t: NeighborTable, p: HalgrenParams,
                       exclude: bool = False) -> ForceAccumulator:
        fx, fy, fz = self._vec3()
        e = C.c_double()
        w = np.zeros(9)
        check(self.lib.mdg_halgren_forces(self.ctx, t.list_id, p.cutoff, p.delta, p.gamma,
                                          int(exclude), _p(fx), _p(fy), _p(fz), C.byref(e),
                                          _p(w)))
        return ForceAccumulator(fx, fy, fz, e.value, w.reshape(3, 3))

    def dipole_field_matvec(self, t: NeighborTable, state: PolarizationState, p: PolarParams,
                            alpha: float = 0.0) -> FieldArrays:
        mx, my, mz = _f64(state.mu_x), _f64(state.mu_y), _f64(state.mu_z)
        ex, ey, ez = self._vec3()
        # the reference mat-vec reads state.thole_a (proj/src/polar_scalar.cpp:79)
        check(self.lib.mdg_tmatvec(self.ctx, t.list_id, alpha, p.cutoff, state.thole_a, _p(mx),
                                   _p(my), _p(mz), _p(ex), _p(ey), _p(ez)))
        return FieldArrays(ex, ey, ez)

    def permanent_field(self, t: NeighborTable, p: PolarParams, alpha: float = 0.0,
                        exclude: bool = False) -> FieldArrays:
        ex, ey, ez = self._vec3()
        check(self.lib.mdg_perm_field(self.ctx, t.list_id, alpha, p.cutoff, p.thole_a,
                                      int(exclude), _p(ex), _p(ey), _p(ez)))
        return FieldArrays(ex, ey, ez)

    def jacobi_polarization_solve(self, t: NeighborTable, p: PolarParams, tol: float,
                                  max_iter: int) -> PolarizationState:
        mx, my, mz = self._vec3()
        it, res = C.c_int64(), C.c_double()
        rc = self.lib.mdg_polar_solve_jacobi(self.ctx, t.list_id, p.cutoff, p.thole_a, tol,
                                             int(max_iter), _p(mx), _p(my), _p(mz),
                                             C.byref(it), C.byref(res))
        check(rc, res.value)
        return PolarizationState(mx, my, mz, p.thole_a, it.value, res.value)

    def polar_solve_pcg(self, t: NeighborTable, p: PolarParams, alpha: float = 0.0,
                        tol_debye: float = 1e-5, max_iter: int = 100,
                        exclude_perm: bool = False) -> PolarizationState:
        mx, my, mz = self._vec3()
        it, rms = C.c_int64(), C.c_double()
        rc = self.lib.mdg_polar_solve_pcg(self.ctx, t.list_id, alpha, p.cutoff, p.thole_a,
                                          int(exclude_perm), tol_debye, int(max_iter), _p(mx),
                                          _p(my), _p(mz), C.byref(it), C.byref(rms))
        check(rc, rms.value)
        return PolarizationState(mx, my, mz, p.thole_a, it.value, rms.value)

    def mpole_forces(self, t: NeighborTable, alpha: float, cutoff: float, electric: float = 1.0,
                     exclude: bool = True):
        fx, fy, fz = self._vec3()
        tx, ty, tz = self._vec3()
        e = C.c_double()
        w = np.zeros(9)
        check(self.lib.mdg_mpole_forces(self.ctx, t.list_id, alpha, cutoff, electric,
                                        int(exclude), _p(fx), _p(fy), _p(fz), _p(tx), _p(ty),
                                        _p(tz), C.byref(e), _p(w)))
        return (_aos(fx, fy, fz), _aos(tx, ty, tz), e.value, w.reshape(3, 3))

    def polar_forces(self, t: NeighborTable, p: "PolarParams", alpha: float,
                     electric: float = 1.0, mu=None, exclude: bool = True):
        """Polarization forces, torques on the permanent multipoles, pair
        energy and pair virial at dipoles mu ((n, 3), caller order; None = the
        context's last solve). mdg.h mdg_polar_forces."""
        fx, fy, fz = self._vec3()
        tx, ty, tz = self._vec3()
        e = C.c_double()
        w = np.zeros(9)
        mx = my = mz = None
        if mu is not None:
            mu = np.asarray(mu, np.float64)
            mx, my, mz = _f64(mu[:, 0]), _f64(mu[:, 1]), _f64(mu[:, 2])
        check(self.lib.mdg_polar_forces(self.ctx, t.list_id, alpha, p.cutoff, p.thole_a,
                                        electric, int(exclude), _p(mx), _p(my), _p(mz), _p(fx),
                                        _p(fy), _p(fz), _p(tx), _p(ty), _p(tz), C.byref(e),
                                        _p(w)))
        return (_aos(fx, fy, fz), _aos(tx, ty, tz), e.value, w.reshape(3, 3))

    def ewald_recip(self, alpha: float, grid=(32, 32, 32), order: int = 5,
                    electric: float = 1.0, exclude: bool = True):
        """Smooth-PME reciprocal space (mdg.h mdg_ewald_recip): (forces,
        (E_recip, E_self, E_excluded), virial 3x3)."""
        fx, fy, fz = self._vec3()
        e = np.zeros(3)
        w = np.zeros(9)
        check(self.lib.mdg_ewald_recip(self.ctx, alpha, int(grid[0]), int(grid[1]), int(grid[2]),
                                       int(order), electric, int(exclude), _p(fx), _p(fy),
                                       _p(fz), _p(e), _p(w)))
        return _aos(fx, fy, fz), e, w.reshape(3, 3)

    # ---- MD (8(f)#4) ---------------------------------------------------------------
    def resort(self):
        """Re-sort the sites spatially on the device (mdg_resort); lists must
        be rebuilt afterwards."""
        check(self.lib.mdg_resort(self.ctx))

    def set_ewald_recip(self, grid=(0, 0, 0), order: int = 6):
        """Reciprocal-space Ewald in amoeba_step / polar_solve_pcg
        (mdg_set_ewald_recip); grid (0, 0, 0) switches it off."""
        check(self.lib.mdg_set_ewald_recip(self.ctx, *map(int, grid), int(order)))

    def ewald_recip_mpole(self, alpha: float, grid=(48, 48, 48), order: int = 6,
                          electric: float = 1.0, exclude: bool = True):
        """Smooth PME of the permanent multipoles: (forces, torques,
        (E_recip, E_self, E_excluded)) -- mdg_ewald_recip_mpole."""
        fx, fy, fz = self._vec3()
        tx, ty, tz = self._vec3()
        e = np.zeros(3)
        check(self.lib.mdg_ewald_recip_mpole(self.ctx, float(alpha), *map(int, grid), int(order),
                                             float(electric), int(exclude), _p(fx), _p(fy),
                                             _p(fz), _p(tx), _p(ty), _p(tz), _p(e)))
        return np.stack([fx, fy, fz], 1), np.stack([tx, ty, tz], 1), e

    def upload_bonded(self, bonds=None, kb=None, r0=None, angles=None, ka=None, theta0=None):
        """Harmonic bonds (m, 2) / angles (m, 3; vertex in the middle),
        E = k (x - x0)^2 (mdg.h mdg_bonded_upload)."""
        b = np.zeros((0, 2), np.int32) if bonds is None else np.ascontiguousarray(bonds, np.int32)
        a = np.zeros((0, 3), np.int32) if angles is None else np.ascontiguousarray(angles, np.int32)
        kb_ = _f64(np.zeros(0) if kb is None else np.broadcast_to(kb, len(b)))
        r0_ = _f64(np.zeros(0) if r0 is None else np.broadcast_to(r0, len(b)))
        ka_ = _f64(np.zeros(0) if ka is None else np.broadcast_to(ka, len(a)))
        t0_ = _f64(np.zeros(0) if theta0 is None else np.broadcast_to(theta0, len(a)))
        check(self.lib.mdg_bonded_upload(self.ctx, len(b), _p(b, _ip), _p(kb_), _p(r0_), len(a),
                                         _p(a, _ip), _p(ka_), _p(t0_)))

    def bonded_forces(self):
        fx, fy, fz = self._vec3()
        e = np.zeros(2)
        check(self.lib.mdg_bonded_forces(self.ctx, _p(fx), _p(fy), _p(fz), _p(e)))
        return _aos(fx, fy, fz), e

    def upload_velocities(self, v, mass=None):
        v = np.asarray(v, np.float64)
        vx, vy, vz = _f64(v[:, 0]), _f64(v[:, 1]), _f64(v[:, 2])
        m = None if mass is None else _f64(mass)
        check(self.lib.mdg_velocities_upload(self.ctx, _p(m), _p(vx), _p(vy), _p(vz)))

    def fetch_velocities(self) -> np.ndarray:
        vx, vy, vz = self._vec3()
        check(self.lib.mdg_velocities_fetch(self.ctx, _p(vx), _p(vy), _p(vz)))
        return _aos(vx, vy, vz)

    def fetch_positions(self) -> np.ndarray:
        x, y, z = self._vec3()
        check(self.lib.mdg_positions_fetch(self.ctx, _p(x), _p(y), _p(z)))
        return _aos(x, y, z)

    def md_run(self, p: "MDParams", charmm=None, amoeba=None, energies: bool = True):
        """Velocity Verlet or BAOAB-RESPA on the device (mdg.h mdg_md_run);
        returns per-step (kinetic, potential) energies when `energies`."""
        ek = np.zeros(max(p.nsteps, 1)) if energies else None
        ep = np.zeros(max(p.nsteps, 1)) if energies else None
        check(self.lib.mdg_md_run(self.ctx, C.byref(p), None if charmm is None else C.byref(charmm),
                                  None if amoeba is None else C.byref(amoeba), _p(ek), _p(ep)))
        return (ek[: p.nsteps], ep[: p.nsteps]) if energies else None

    def md_rebuild_count(self) -> int:
        """List rebuilds done by md_run so far (mdg_md_rebuild_count)."""
        v = C.c_int64()
        check(self.lib.mdg_md_rebuild_count(self.ctx, C.byref(v)))
        return v.value

    # ---- fused steps ----------------------------------------------------------------
    def charmm_step(self, t: NeighborTable, p: CharmmParams):
        check(self.lib.mdg_charmm_step(self.ctx, t.list_id, C.byref(p)))

    def amoeba_step(self, vdw: NeighborTable, elec: NeighborTable, p: AmoebaParams):
        check(self.lib.mdg_amoeba_step(self.ctx, vdw.list_id, elec.list_id, C.byref(p)))

    def fetch_forces(self, out=None) -> np.ndarray:
        """(n, 3) forces; `out` = an optional (3, n) float64 block (e.g. a
        host_array, which is filled by DMA without a staging copy)."""
        if out is None:
            fx, fy, fz = self._vec3()
        else:
            assert out.shape == (3, self.n) and out.dtype == np.float64 and out.flags.c_contiguous
            fx, fy, fz = out[0], out[1], out[2]
        check(self.lib.mdg_fetch_forces(self.ctx, _p(fx), _p(fy), _p(fz)))
        return _aos(fx, fy, fz)

    def set_force_output(self, out=None):
        """Register a (3, n) page-locked block (host_array) that every later
        step fills with its forces by DMA, overlapped with the rest of the
        step (mdg.h mdg_set_force_output); fetch_forces(out=that block) then
        only waits. None unregisters."""
        if out is None:
            check(self.lib.mdg_set_force_output(self.ctx, None, None, None))
            self._fout = None
            return
        assert out.shape == (3, self.n) and out.dtype == np.float64 and out.flags.c_contiguous
        check(self.lib.mdg_set_force_output(self.ctx, _p(out[0]), _p(out[1]), _p(out[2])))
        self._fout = out  # keep the buffer alive while registered

    def fetch_torques(self) -> np.ndarray:
        tx, ty, tz = self._vec3()
        check(self.lib.mdg_fetch_torques(self.ctx, _p(tx), _p(ty), _p(tz)))
        return _aos(tx, ty, tz)

    def fetch_dipoles(self) -> np.ndarray:
        mx, my, mz = self._vec3()
        check(self.lib.mdg_fetch_dipoles(self.ctx, _p(mx), _p(my), _p(mz)))
        return _aos(mx, my, mz)

    def fetch_perm_field(self) -> np.ndarray:
        ex, ey, ez = self._vec3()
        check(self.lib.mdg_fetch_perm_field(self.ctx, _p(ex), _p(ey), _p(ez)))
        return _aos(ex, ey, ez)

    def fetch_energies(self):
        e = np.zeros(4)
        w = np.zeros(9)
        it, rms = C.c_int64(), C.c_double()
        check(self.lib.mdg_fetch_energies(self.ctx, _p(e), _p(w), C.byref(it), C.byref(rms)))
        return e, w.reshape(3, 3), it.value, rms.value

    def synchronize(self):
        check(self.lib.mdg_ctx_synchronize(self.ctx))

    def stream(self) -> int:
        return self.lib.mdg_ctx_stream(self.ctx) or 0

    def count_within(self, t: NeighborTable, cutoff: float, exclude: bool = False):
        """(directed pairs within cutoff, list slots) of a device list."""
        a, b = C.c_int64(), C.c_int64()
        check(self.lib.mdg_nlist_count_within(self.ctx, t.list_id, cutoff, int(exclude),
                                              C.byref(a), C.byref(b)))
        return a.value, b.value

    # ---- instrumentation -------------------------------------------------------------
    def timer_start(self):
        check(self.lib.mdg_timer_start(self.ctx))

    def timer_stop(self) -> float:
        """Device milliseconds since timer_start (CUDA events on the ctx stream)."""
        ms = C.c_double()
        check(self.lib.mdg_timer_stop(self.ctx, C.byref(ms)))
        return ms.value

    def upload_frames(self, frame_type, zatom, xatom, dipole=None, quadrupole=None):
        """Local multipole frames (mdg.h mdg_frames_upload): type 0 none,
        1 z-then-x, 2 bisector; dipole (n, 3) / quadrupole (n, 6) in the
        local frames. frame_type None removes the frames."""
        if frame_type is None:
            check(self.lib.mdg_frames_upload(self.ctx, None, None, None, None, None))
            return
        t = np.ascontiguousarray(frame_type, np.int32)
        z = np.ascontiguousarray(zatom, np.int32)
        x = np.ascontiguousarray(xatom, np.int32)
        d = None if dipole is None else _f64(np.asarray(dipole).reshape(-1))
        q = None if quadrupole is None else _f64(np.asarray(quadrupole).reshape(-1))
        check(self.lib.mdg_frames_upload(self.ctx, _p(t, _ip), _p(z, _ip), _p(x, _ip), _p(d),
                                         _p(q)))

    def set_deterministic(self, on: bool = True):
        """Full-row pair sums (bitwise reproducible forces/torques) instead of
        the default half rows with atomic partner updates (mdg.h)."""
        check(self.lib.mdg_set_deterministic(self.ctx, int(on)))

    def set_debug_perturb(self, delta: float = 0.0):
        """Fault injection (reference debug_perturb_vectorized): delta added to
        the first returned force component and energy."""
        check(self.lib.mdg_set_debug_perturb(self.ctx, float(delta)))

    def set_overlap(self, on: bool = True):
        """AMOEBA step on two streams (default) or one (mdg.h)."""
        check(self.lib.mdg_set_overlap(self.ctx, int(on)))

    def set_cluster_matvec(self, on: bool = True):
        """PCG mat-vec on 3-site clusters (opt-in) or per-site rows (mdg.h)."""
        check(self.lib.mdg_set_cluster_matvec(self.ctx, int(on)))

    def set_cluster_halgren(self, on: bool = True):
        """Halgren on 3-site clusters (default) or per-site half rows (mdg.h)."""
        check(self.lib.mdg_set_cluster_halgren(self.ctx, int(on)))

    def launch_count(self) -> int:
        return int(self.lib.mdg_launch_count(self.ctx))

    def profile(self, enable: bool):
        check(self.lib.mdg_profile_enable(self.ctx, int(enable)))

    def profile_reset(self):
        check(self.lib.mdg_profile_reset(self.ctx))

    def profile_report(self) -> dict:
        buf = C.create_string_buffer(1 << 16)
        check(self.lib.mdg_profile_report(self.ctx, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split()
            out[name] = (int(cnt), float(ms))
        return out


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured FP64 DFMA peak of the device (TFLOP/s)."""
    v = C.c_double()
    check(load_library().mdg_probe_fp64_peak(device, C.byref(v)))
    return v.value


class _Pinned:
    """Owner of one page-locked allocation (freed with the last view)."""

    def __init__(self, nbytes: int):
        self.lib = load_library()
        self.ptr = C.c_void_p()
        check(self.lib.mdg_host_alloc(C.byref(self.ptr), nbytes))

    def __del__(self):
        if self.ptr:
            self.lib.mdg_host_free(self.ptr)
            self.ptr = C.c_void_p()


def host_array(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (mdg_host_alloc): per-step
    coordinates / results kept here are DMA'd without a staging copy."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape))
    owner = _Pinned(max(1, n * dt.itemsize))
    buf = (C.c_char * max(1, n * dt.itemsize)).from_address(owner.ptr.value)
    buf._owner = owner  # the array's base keeps the allocation alive
    return np.frombuffer(buf, dtype=dt, count=n).reshape(shape)


def device_erfc(x, device: int = 0) -> np.ndarray:
    """The pair kernels' erfc evaluated on the device (accuracy probe)."""
    x = _f64(x)
    out = np.zeros_like(x)
    check(load_library().mdg_probe_erfc(device, _p(x), len(x), _p(out)))
    return out


# ---- the reference's system dump format (interop) --------------------------------
_JSON_ARRAYS = ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
                "polarizability")


def load_system_json(path_or_text: str):
    """Read the reference's `bench gen` system dump (mdvec::dump_system_json,
    proj/src/bench.cpp:541-567: version, seed, kind, box, n_sites, the nine
    site arrays, mu_x/mu_y/mu_z). Returns (ParticleSystem, dipoles (n, 3) or
    None, metadata dict)."""
    import json
    import os
    text = path_or_text
    if not text.lstrip().startswith("{") and os.path.exists(path_or_text):
        with open(path_or_text) as f:
            text = f.read()
    j = json.loads(text)
    if j.get("version") != 1:
        raise ContractViolation("system dump: unsupported version %r" % j.get("version"))
    n = int(j["n_sites"])
    arrs = {}
    for k in _JSON_ARRAYS:
        a = np.asarray(j[k], np.float64)
        if a.shape != (n,):
            raise ContractViolation(f"system dump: {k} has {a.shape[0]} values, expected {n}")
        arrs[k] = a
    b = j["box"]
    s = ParticleSystem((float(b["lx"]), float(b["ly"]), float(b["lz"])), **arrs)
    mu = None
    if all(k in j for k in ("mu_x", "mu_y", "mu_z")):
        mu = np.stack([np.asarray(j[k], np.float64) for k in ("mu_x", "mu_y", "mu_z")], 1)
    meta = {k: j[k] for k in ("version", "seed", "kind") if k in j}
    return s, mu, meta


def dump_system_json(s, mu=None, seed: int = 1, kind: str = "uniform-random") -> str:
    """The same format, written from a ParticleSystem (+ optional dipoles)."""
    import json
    j = {"version": 1, "seed": int(seed), "kind": kind,
         "box": {"lx": float(s.box[0]), "ly": float(s.box[1]), "lz": float(s.box[2])},
         "n_sites": int(len(s.x))}
    for k in _JSON_ARRAYS:
        j[k] = [float(v) for v in np.asarray(getattr(s, k), np.float64)]
    if mu is not None:
        mu = np.asarray(mu, np.float64)
        for a, k in enumerate(("mu_x", "mu_y", "mu_z")):
            j[k] = [float(v) for v in mu[:, a]]
    return json.dumps(j, indent=2, sort_keys=True) + "\n"


# ---- fixtures ------------------------------------------------------------------------
def water_box(n_mol: int, box: float, seed: int = 1, model: str = "amoeba") -> ParticleSystem:
    """BASELINE.json 3-site water fixture (mdg_water_generate)."""
    lib = load_library()
    n = 3 * n_mol
    f = {k: np.zeros(n) for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0",
                                  "hal_epsilon", "polarizability", "hred_factor")}
    mol = np.zeros(n, np.int32)
    par = np.zeros(n, np.int32)
    dip = np.zeros(3 * n)
    quad = np.zeros(6 * n)
    rc = lib.mdg_water_generate(n_mol, box, seed, 0 if model == "charmm" else 1,
                                _p(f["x"]), _p(f["y"]), _p(f["z"]), _p(mol, _ip),
                                _p(f["charge"]), _p(f["lj_sigma"]), _p(f["lj_epsilon"]),
                                _p(f["hal_r0"]), _p(f["hal_epsilon"]), _p(f["polarizability"]),
                                _p(par, _ip), _p(f["hred_factor"]), _p(dip), _p(quad))
    check(rc)
    amoeba = model != "charmm"
    return ParticleSystem((box, box, box), f["x"], f["y"], f["z"], f["charge"], f["lj_sigma"],
                          f["lj_epsilon"], f["hal_r0"], f["hal_epsilon"], f["polarizability"],
                          molecule=mol,
                          dipole=dip.reshape(n, 3) if amoeba else None,
                          quadrupole=quad.reshape(n, 6) if amoeba else None,
                          hred_parent=par if amoeba else None,
                          hred_factor=f["hred_factor"] if amoeba else None)


def reduce_sites_host(s) -> tuple:
    """Halgren-reduced coordinates, bit-identical to the device's."""
    lib = load_library()
    n = s.n_sites if hasattr(s, "n_sites") else len(s.x)
    out = [np.zeros(n) for _ in range(3)]
    par = np.ascontiguousarray(s.hred_parent, np.int32)
    fac = _f64(s.hred_factor)
    check(lib.mdg_reduce_sites_host(n, *map(float, s.box), _p(_f64(s.x)), _p(_f64(s.y)),
                                    _p(_f64(s.z)), _p(par, _ip), _p(fac), *(_p(v) for v in out)))
    return tuple(out)


# configuration table from BASELINE.json
CONFIGS = {
    0: dict(n_mol=1000, box=31.04, model="charmm", cutoff=9.0, skin=2.0, alpha=0.35),
    1: dict(n_mol=8000, box=62.1, model="amoeba", vdw_cutoff=9.0, elec_cutoff=7.0, skin=2.0,
            alpha=0.5446),
    2: dict(n_mol=8000, box=62.1, model="amoeba", vdw_cutoff=9.0, elec_cutoff=7.0, skin=2.0,
            alpha=0.5446),
    3: dict(n_mol=32000, box=98.6, model="amoeba", vdw_cutoff=9.0, elec_cutoff=7.0, skin=2.0,
            alpha=0.5446),
    4: dict(n_mol=333333, box=215.3, model="amoeba", vdw_cutoff=9.0, elec_cutoff=7.0, skin=2.0,
            alpha=0.5446, rebuild_every=20),
}
