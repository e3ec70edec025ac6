"""ctypes front-end for the CHECKERS (test infrastructure only).

`Oracle` wraps liboracle.so (the plain-C restatement, mdo.c) and `RefLib`
wraps oracle/_ref/libmdvec_ref_<isa>.so (the unmodified reference library
plus ref_shim.cpp). Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / --impl reference legs import this module. The product package
(paper_1906_01211_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint32)
_lp = C.POINTER(C.c_uint64)

STATUS_NAMES = {1: "ContractViolation", 2: "CapacityError", 3: "SingularityError",
                4: "ConvergenceError", 5: "GenerationError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _ptr(a, t=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so with gcc if it is missing (the GPU box has gcc)."""
    so = os.path.join(HERE, "liboracle.so")
    src = os.path.join(HERE, "mdo.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    return so


class MdoSystem(C.Structure):
    _fields_ = [("n", C.c_size_t), ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("x", _dp), ("y", _dp), ("z", _dp), ("charge", _dp), ("lj_sigma", _dp),
                ("lj_epsilon", _dp), ("hal_r0", _dp), ("hal_epsilon", _dp),
                ("polarizability", _dp), ("molecule", _ip), ("dipole", _dp),
                ("quadrupole", _dp)]


class MdoTable(C.Structure):
    _fields_ = [("n_sites", C.c_size_t), ("cutoff", C.c_double), ("nnvlst", _up),
                ("nvloop8", _up), ("nvloop16", _up), ("offset", _lp), ("indices", _ip),
                ("scale", _dp), ("total", C.c_size_t)]


@dataclass
class System:
    """Plain-array site data in the reference's (original) order."""
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
    dipole: np.ndarray | None = None       # (n, 3)
    quadrupole: np.ndarray | None = None   # (n, 6) xx,xy,xz,yy,yz,zz
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n(self) -> int:
        return int(self.x.shape[0])

    def copy(self) -> "System":
        kw = {k: (None if getattr(self, k) is None else np.array(getattr(self, k)))
              for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0",
                        "hal_epsilon", "polarizability", "molecule", "dipole", "quadrupole")}
        return System(box=tuple(self.box), **kw)

    def as_struct(self) -> MdoSystem:
        arrs = {}
        for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
                  "polarizability"):
            arrs[k] = np.ascontiguousarray(getattr(self, k), dtype=np.float64)
        mol = None if self.molecule is None else np.ascontiguousarray(self.molecule, np.int32)
        dip = None if self.dipole is None else np.ascontiguousarray(self.dipole, np.float64)
        quad = None if self.quadrupole is None else np.ascontiguousarray(self.quadrupole,
                                                                         np.float64)
        self._keep = [arrs, mol, dip, quad]
        return MdoSystem(self.n, float(self.box[0]), float(self.box[1]), float(self.box[2]),
                         *(_ptr(arrs[k]) for k in ("x", "y", "z", "charge", "lj_sigma",
                                                   "lj_epsilon", "hal_r0", "hal_epsilon",
                                                   "polarizability")),
                         _ptr(mol, _ip), _ptr(dip), _ptr(quad))


@dataclass
class Table:
    """Reference NeighborTable layout (proj/include/mdvec/neighbors.hpp:25-41)."""
    cutoff: float
    nnvlst: np.ndarray
    nvloop8: np.ndarray
    nvloop16: np.ndarray
    offset: np.ndarray
    indices: np.ndarray
    scale: np.ndarray

    @property
    def n_sites(self) -> int:
        return int(self.nnvlst.shape[0])

    def pairs(self) -> np.ndarray:
        """table_pairs(): canonical (i<j) lexicographically sorted pairs."""
        rows = []
        for i in range(self.n_sites):
            j = self.indices[self.offset[i]: self.offset[i] + self.nnvlst[i]].astype(np.int64)
            rows.append(np.stack([np.minimum(i, j), np.maximum(i, j)], 1))
        p = np.concatenate(rows) if rows else np.zeros((0, 2), np.int64)
        return sort_pairs(p)

    def filtered(self, molecule: np.ndarray) -> "Table":
        """Drop same-molecule j from each segment and re-pad."""
        nn, nv8, nv16, off, idx = [], [], [], [], []
        pos = 0
        for i in range(self.n_sites):
            seg = self.indices[self.offset[i]: self.offset[i] + self.nnvlst[i]]
            seg = seg[molecule[seg] != molecule[i]]
            k = len(seg)
            p16 = (k + 15) & ~15
            nn.append(k)
            nv8.append((k + 7) & ~7)
            nv16.append(p16)
            off.append(pos)
            sent = seg[-1] if k else 0
            idx.append(np.concatenate([seg, np.full(p16 - k, sent, np.int32)]))
            pos += p16
        indices = np.concatenate(idx).astype(np.int32) if idx else np.zeros(0, np.int32)
        scale = np.zeros(len(indices))
        for i in range(self.n_sites):
            scale[off[i]: off[i] + nn[i]] = 1.0
        return Table(self.cutoff, np.array(nn, np.uint32), np.array(nv8, np.uint32),
                     np.array(nv16, np.uint32), np.array(off, np.uint64), indices, scale)

    def as_struct(self) -> MdoTable:
        self._keep = [np.ascontiguousarray(a) for a in
                      (self.nnvlst, self.nvloop8, self.nvloop16, self.offset, self.indices,
                       self.scale)]
        k = self._keep
        return MdoTable(self.n_sites, self.cutoff, _ptr(k[0], _up), _ptr(k[1], _up),
                        _ptr(k[2], _up), _ptr(k[3], _lp), _ptr(k[4], _ip), _ptr(k[5]),
                        int(self.indices.shape[0]))


def sort_pairs(p: np.ndarray) -> np.ndarray:
    p = np.asarray(p, np.int64).reshape(-1, 2)
    if len(p) == 0:
        return p
    order = np.lexsort((p[:, 1], p[:, 0]))
    return p[order]


class Oracle:
    """The plain-C restatement (mdo.c)."""

    def __init__(self, path: str | None = None):
        self.lib = C.CDLL(path or build_oracle())
        L = self.lib
        L.mdo_last_error.restype = C.c_char_p
        L.mdo_wrap1.restype = C.c_double
        L.mdo_wrap1.argtypes = [C.c_double] * 4
        L.mdo_dist2.restype = C.c_double
        L.mdo_dist2.argtypes = [C.c_double] * 3
        L.mdo_table_build.argtypes = [C.POINTER(MdoSystem), C.c_double, C.c_size_t,
                                      C.POINTER(MdoTable)]
        L.mdo_table_free.argtypes = [C.POINTER(MdoTable)]
        L.mdo_generate_system.argtypes = [C.c_int, C.c_size_t, C.c_double, C.c_double,
                                          C.c_double, C.c_uint64, C.c_double] + [_dp] * 9
        L.mdo_random_dipoles.argtypes = [C.c_size_t, C.c_uint64, C.c_double, _dp, _dp, _dp]
        L.mdo_brute_force_pairs.argtypes = [C.POINTER(MdoSystem), C.c_double, _ip, C.c_size_t,
                                            C.POINTER(C.c_size_t)]
        L.mdo_ewald_bn.argtypes = [C.c_double, C.c_double, C.c_int, _dp]
        L.mdo_reduce_sites.argtypes = [C.c_size_t, _dp, _dp, _dp, _ip, _dp, C.c_double,
                                       C.c_double, C.c_double, _dp, _dp, _dp]
        L.mdo_reduce_forces.argtypes = [C.c_size_t, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.mdo_rows_for_sites.argtypes = [C.POINTER(MdoSystem), C.c_double, _ip, C.c_size_t, _ip,
                                         _ip, C.c_size_t]
        L.mdo_water_generate.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.c_int, _dp, _dp,
                                         _dp, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _dp, _dp,
                                         _dp]

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.mdo_last_error().decode())

    # -- geometry
    def wrap1(self, d, L):
        return self.lib.mdo_wrap1(d, L, 1.0 / L, 0.5 * L)

    def minimum_image(self, d, box):
        return tuple(self.wrap1(d[a], box[a]) for a in range(3))

    # -- reference generator restatement
    def generate_system(self, kind: str, n: int, box, seed: int, min_sep: float = 0.8) -> System:
        arrs = [np.zeros(n) for _ in range(9)]
        k = 0 if kind == "lattice" else 1
        self._check(self.lib.mdo_generate_system(k, n, *map(float, box), seed, min_sep,
                                                 *(_ptr(a) for a in arrs)))
        return System(tuple(map(float, box)), *arrs)

    def water_box(self, n_mol: int, box: float, seed: int = 1, model: str = "amoeba"):
        """BASELINE.json 3-site water fixture (mdo_water_generate, the oracle's
        own restatement; bit-identical to the product's mdg_water_generate,
        tests/test_oracle.py). Returns (System, hred_parent, hred_factor)."""
        n = 3 * n_mol
        f = {k: np.zeros(n) for k in ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon",
                                      "hal_r0", "hal_epsilon", "polarizability", "hred_factor")}
        mol = np.zeros(n, np.int32)
        par = np.zeros(n, np.int32)
        dip = np.zeros(3 * n)
        quad = np.zeros(6 * n)
        self._check(self.lib.mdo_water_generate(
            n_mol, box, seed, 0 if model == "charmm" else 1, _ptr(f["x"]), _ptr(f["y"]),
            _ptr(f["z"]), _ptr(mol, _ip), _ptr(f["charge"]), _ptr(f["lj_sigma"]),
            _ptr(f["lj_epsilon"]), _ptr(f["hal_r0"]), _ptr(f["hal_epsilon"]),
            _ptr(f["polarizability"]), _ptr(par, _ip), _ptr(f["hred_factor"]), _ptr(dip),
            _ptr(quad)))
        amoeba = model != "charmm"
        s = System((box, box, box), f["x"], f["y"], f["z"], f["charge"], f["lj_sigma"],
                   f["lj_epsilon"], f["hal_r0"], f["hal_epsilon"], f["polarizability"],
                   molecule=mol, dipole=dip.reshape(n, 3) if amoeba else None,
                   quadrupole=quad.reshape(n, 6) if amoeba else None)
        return s, par, f["hred_factor"]

    def random_dipoles(self, n: int, seed: int, magnitude: float = 0.1) -> np.ndarray:
        a = [np.zeros(n) for _ in range(3)]
        self.lib.mdo_random_dipoles(n, seed, magnitude, *(_ptr(v) for v in a))
        return np.stack(a, 1)

    # -- neighbour table
    def build_table(self, s: System, list_cutoff: float, extra_pad: int = 0) -> Table:
        st = s.as_struct()
        t = MdoTable()
        self._check(self.lib.mdo_table_build(C.byref(st), list_cutoff, extra_pad, C.byref(t)))
        n = t.n_sites
        try:
            return Table(t.cutoff,
                         np.ctypeslib.as_array(t.nnvlst, (n,)).copy() if n else np.zeros(0, np.uint32),
                         np.ctypeslib.as_array(t.nvloop8, (n,)).copy() if n else np.zeros(0, np.uint32),
                         np.ctypeslib.as_array(t.nvloop16, (n,)).copy() if n else np.zeros(0, np.uint32),
                         np.ctypeslib.as_array(t.offset, (n,)).copy() if n else np.zeros(0, np.uint64),
                         np.ctypeslib.as_array(t.indices, (t.total,)).copy() if t.total else np.zeros(0, np.int32),
                         np.ctypeslib.as_array(t.scale, (t.total,)).copy() if t.total else np.zeros(0))
        finally:
            self.lib.mdo_table_free(C.byref(t))

    def rows_for_sites(self, s: System, cutoff: float, sites) -> list:
        """Full rows (all j != i within cutoff, ascending) of `sites`, brute
        force with the reference predicate (mdo_rows_for_sites)."""
        sites = np.ascontiguousarray(sites, np.int32)
        st = s.as_struct()
        counts = np.zeros(len(sites), np.int32)
        vol = float(np.prod(s.box))
        cap = int(len(sites) * (s.n / vol * 4.2 * cutoff ** 3 * 2 + 64))
        idx = np.zeros(cap, np.int32)
        self._check(self.lib.mdo_rows_for_sites(C.byref(st), cutoff, _ptr(sites, _ip), len(sites),
                                                _ptr(counts, _ip), _ptr(idx, _ip), cap))
        ends = np.cumsum(counts)
        return [idx[e - c:e].copy() for c, e in zip(counts, ends)]

    @staticmethod
    def table_from_rows(n: int, cutoff: float, sites, rows) -> Table:
        """A reference-layout table whose only non-empty segments are the given
        rows (segment of sites[k] = rows[k], padded to 16 with the sentinel)."""
        nn = np.zeros(n, np.uint32)
        nn[np.asarray(sites)] = [len(r) for r in rows]
        p16 = (nn.astype(np.int64) + 15) & ~15
        off = np.zeros(n, np.uint64)
        off[1:] = np.cumsum(p16)[:-1]
        idx = np.zeros(int(p16.sum()), np.int32)
        scale = np.zeros(len(idx))
        for site, r in zip(sites, rows):
            o = int(off[site])
            k = len(r)
            idx[o:o + k] = r
            idx[o + k:o + int(p16[site])] = r[-1] if k else 0
            scale[o:o + k] = 1.0
        nv8 = ((nn.astype(np.int64) + 7) & ~7).astype(np.uint32)
        return Table(cutoff, nn, nv8, p16.astype(np.uint32), off, idx, scale)

    def brute_force_pairs(self, s: System, cutoff: float) -> np.ndarray:
        st = s.as_struct()
        cap = 1 << 16
        while True:
            out = np.zeros(2 * cap, np.int32)
            npairs = C.c_size_t()
            rc = self.lib.mdo_brute_force_pairs(C.byref(st), cutoff, _ptr(out, _ip), cap,
                                                C.byref(npairs))
            if rc == 2:
                cap = npairs.value
                continue
            self._check(rc)
            return out[: 2 * npairs.value].reshape(-1, 2).astype(np.int64)

    # -- kernels
    def _forces(self, fn, s, t, *args, exclude=False):
        n = s.n
        st, tt = s.as_struct(), t.as_struct()
        fx, fy, fz = np.zeros(n), np.zeros(n), np.zeros(n)
        e = C.c_double()
        w = np.zeros(9)
        self._check(fn(C.byref(st), C.byref(tt), *args, int(exclude), _ptr(fx), _ptr(fy),
                       _ptr(fz), C.byref(e), _ptr(w)))
        return np.stack([fx, fy, fz], 1), e.value, w.reshape(3, 3)

    def lj(self, s, t, cutoff, shift=False, exclude=False):
        return self._forces(self.lib.mdo_lj, s, t, C.c_double(cutoff), C.c_int(int(shift)),
                            exclude=exclude)

    def ewald_real(self, s, t, alpha, cutoff, electric=1.0, exclude=False):
        return self._forces(self.lib.mdo_ewald_real, s, t, C.c_double(alpha), C.c_double(cutoff),
                            C.c_double(electric), exclude=exclude)

    def halgren(self, s, t, cutoff, delta=0.07, gamma=0.12, exclude=False):
        return self._forces(self.lib.mdo_halgren, s, t, C.c_double(cutoff), C.c_double(delta),
                            C.c_double(gamma), exclude=exclude)

    def tmatvec_thole(self, s, t, cutoff, thole_a, mu):
        st, tt = s.as_struct(), t.as_struct()
        mu = np.ascontiguousarray(mu, np.float64)
        m = [np.ascontiguousarray(mu[:, a]) for a in range(3)]
        e = [np.zeros(s.n) for _ in range(3)]
        self._check(self.lib.mdo_tmatvec_thole(C.byref(st), C.byref(tt), C.c_double(cutoff),
                                               C.c_double(thole_a), *(_ptr(v) for v in m),
                                               *(_ptr(v) for v in e)))
        return np.stack(e, 1)

    def perm_field_thole(self, s, t, cutoff, thole_a):
        st, tt = s.as_struct(), t.as_struct()
        e = [np.zeros(s.n) for _ in range(3)]
        self._check(self.lib.mdo_perm_field_thole(C.byref(st), C.byref(tt), C.c_double(cutoff),
                                                  C.c_double(thole_a), *(_ptr(v) for v in e)))
        return np.stack(e, 1)

    def jacobi(self, s, t, cutoff, thole_a, tol, max_iter):
        st, tt = s.as_struct(), t.as_struct()
        m = [np.zeros(s.n) for _ in range(3)]
        res = C.c_double()
        it = C.c_size_t()
        rc = self.lib.mdo_jacobi(C.byref(st), C.byref(tt), C.c_double(cutoff),
                                 C.c_double(thole_a), C.c_double(tol), C.c_size_t(max_iter),
                                 *(_ptr(v) for v in m), C.byref(res), C.byref(it))
        if rc == 4:
            err = OracleError(rc, self.lib.mdo_last_error().decode())
            err.last_residual = res.value
            raise err
        self._check(rc)
        return np.stack(m, 1), it.value

    def reduce_sites(self, s: System, parent, factor):
        n = s.n
        out = [np.zeros(n) for _ in range(3)]
        parent = np.ascontiguousarray(parent, np.int32)
        factor = np.ascontiguousarray(factor, np.float64)
        self.lib.mdo_reduce_sites(n, _ptr(np.ascontiguousarray(s.x)),
                                  _ptr(np.ascontiguousarray(s.y)),
                                  _ptr(np.ascontiguousarray(s.z)), _ptr(parent, _ip),
                                  _ptr(factor), *map(float, s.box), *(_ptr(v) for v in out))
        return out

    def reduce_forces(self, parent, factor, fred):
        n = fred.shape[0]
        parent = np.ascontiguousarray(parent, np.int32)
        factor = np.ascontiguousarray(factor, np.float64)
        fr = [np.ascontiguousarray(fred[:, a]) for a in range(3)]
        out = [np.zeros(n) for _ in range(3)]
        self.lib.mdo_reduce_forces(n, _ptr(parent, _ip), _ptr(factor), *(_ptr(v) for v in fr),
                                   *(_ptr(v) for v in out))
        return np.stack(out, 1)

    def ewald_bn(self, r, alpha, nmax=5):
        bn = np.zeros(nmax + 1)
        self.lib.mdo_ewald_bn(r, alpha, nmax, _ptr(bn))
        return bn

    def tmatvec_ewald(self, s, t, alpha, cutoff, thole_a, mu):
        st, tt = s.as_struct(), t.as_struct()
        mu = np.ascontiguousarray(mu, np.float64)
        e = np.zeros((s.n, 3))
        self._check(self.lib.mdo_tmatvec_ewald(C.byref(st), C.byref(tt), C.c_double(alpha),
                                               C.c_double(cutoff), C.c_double(thole_a),
                                               _ptr(mu), _ptr(e)))
        return e

    def perm_field_ewald(self, s, t, alpha, cutoff, thole_a, exclude=True):
        st, tt = s.as_struct(), t.as_struct()
        e = np.zeros((s.n, 3))
        self._check(self.lib.mdo_perm_field_ewald(C.byref(st), C.byref(tt), C.c_double(alpha),
                                                  C.c_double(cutoff), C.c_double(thole_a),
                                                  C.c_int(int(exclude)), _ptr(e)))
        return e

    def mpole_field_tensor(self, s, t, alpha, cutoff, exclude=True):
        st, tt = s.as_struct(), t.as_struct()
        e = np.zeros((s.n, 3))
        self._check(self.lib.mdo_mpole_field_tensor(C.byref(st), C.byref(tt), C.c_double(alpha),
                                                    C.c_double(cutoff), C.c_int(int(exclude)),
                                                    _ptr(e)))
        return e

    def mpole(self, s, t, alpha, cutoff, electric=1.0, exclude=True):
        st, tt = s.as_struct(), t.as_struct()
        f = np.zeros((s.n, 3))
        tq = np.zeros((s.n, 3))
        e = C.c_double()
        w = np.zeros(9)
        self._check(self.lib.mdo_mpole(C.byref(st), C.byref(tt), C.c_double(alpha),
                                       C.c_double(cutoff), C.c_double(electric),
                                       C.c_int(int(exclude)), _ptr(f), _ptr(tq), C.byref(e),
                                       _ptr(w)))
        return f, tq, e.value, w.reshape(3, 3)

    def polar_forces(self, s, t, alpha, cutoff, thole_a, mu, electric=1.0, exclude=True):
        """Polarization forces/torques/pair energy/virial at fixed dipoles mu
        (mdo.h mdo_polar_forces; the epolar1 analogue)."""
        st, tt = s.as_struct(), t.as_struct()
        mu = np.ascontiguousarray(mu, np.float64)
        f = np.zeros((s.n, 3))
        tq = np.zeros((s.n, 3))
        e = C.c_double()
        w = np.zeros(9)
        self._check(self.lib.mdo_polar_forces(C.byref(st), C.byref(tt), C.c_double(alpha),
                                              C.c_double(cutoff), C.c_double(thole_a),
                                              C.c_double(electric), C.c_int(int(exclude)),
                                              _ptr(mu), _ptr(f), _ptr(tq), C.byref(e), _ptr(w)))
        return f, tq, e.value, w.reshape(3, 3)

    def pcg(self, s, t, alpha, cutoff, thole_a, eperm, tol_debye=1e-5, max_iter=100):
        st, tt = s.as_struct(), t.as_struct()
        eperm = np.ascontiguousarray(eperm, np.float64)
        mu = np.zeros((s.n, 3))
        it = C.c_size_t()
        rms = C.c_double()
        self._check(self.lib.mdo_pcg(C.byref(st), C.byref(tt), C.c_double(alpha),
                                     C.c_double(cutoff), C.c_double(thole_a), _ptr(eperm),
                                     C.c_double(tol_debye), C.c_size_t(max_iter), _ptr(mu),
                                     C.byref(it), C.byref(rms)))
        return mu, it.value, rms.value


# ---------------------------------------------------------------- reference

def _host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return all(x in flags for x in ("avx512f", "avx512dq", "avx512bw", "avx512vl",
                                        "avx512cd"))
    except OSError:
        return False


def ref_library_path() -> str | None:
    isa = "skylake-avx512" if _host_has_avx512() else "x86-64-v3"
    p = os.path.join(REF_DIR, f"libmdvec_ref_{isa}.so")
    return p if os.path.exists(p) else None


def ref_isa() -> str:
    return "skylake-avx512" if _host_has_avx512() else "x86-64-v3"


class RefLib:
    """The unmodified reference library behind ref_shim.cpp."""

    def __init__(self, path: str | None = None):
        path = path or ref_library_path()
        if path is None:
            raise FileNotFoundError("oracle/_ref not built (make -C oracle ref)")
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_system_create.argtypes = [C.POINTER(C.c_void_p), C.c_size_t, C.c_double,
                                        C.c_double, C.c_double] + [_dp] * 9
        L.ref_system_destroy.argtypes = [C.c_void_p]
        L.ref_generate_system.argtypes = [C.c_int, C.c_size_t, C.c_double, C.c_double,
                                          C.c_double, C.c_uint64, C.c_double] + [_dp] * 9
        L.ref_random_dipoles.argtypes = [C.c_size_t, C.c_uint64, C.c_double, _dp, _dp, _dp]
        L.ref_table_build.argtypes = [C.c_void_p, C.c_double, C.c_size_t, C.c_int,
                                      C.POINTER(C.c_size_t)]
        L.ref_table_set.argtypes = [C.c_void_p, C.c_double, _up, _up, _up, _lp, _ip, C.c_size_t]
        L.ref_table_export.argtypes = [C.c_void_p, _up, _up, _up, _lp, _ip, _dp]
        L.ref_brute_force_pairs.argtypes = [C.c_void_p, C.c_double, _ip, C.c_size_t,
                                            C.POINTER(C.c_size_t)]
        L.ref_forces.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                 C.c_double, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_field.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp,
                                _dp, _dp, _dp, _dp]
        L.ref_jacobi.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_size_t,
                                 _dp, _dp, _dp, _dp]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def generate_system(self, kind: str, n: int, box, seed: int, min_sep: float = 0.8) -> System:
        arrs = [np.zeros(n) for _ in range(9)]
        self._check(self.lib.ref_generate_system(0 if kind == "lattice" else 1, n,
                                                 *map(float, box), seed, min_sep,
                                                 *(_ptr(a) for a in arrs)))
        return System(tuple(map(float, box)), *arrs)

    def random_dipoles(self, n, seed, magnitude=0.1):
        a = [np.zeros(n) for _ in range(3)]
        self.lib.ref_random_dipoles(n, seed, magnitude, *(_ptr(v) for v in a))
        return np.stack(a, 1)

    def handle(self, s: System) -> "RefHandle":
        return RefHandle(self, s)


class RefHandle:
    def __init__(self, ref: RefLib, s: System):
        self.ref, self.n = ref, s.n
        self.h = C.c_void_p()
        arrs = [np.ascontiguousarray(getattr(s, k), np.float64) for k in
                ("x", "y", "z", "charge", "lj_sigma", "lj_epsilon", "hal_r0", "hal_epsilon",
                 "polarizability")]
        ref._check(ref.lib.ref_system_create(C.byref(self.h), s.n, *map(float, s.box),
                                             *(_ptr(a) for a in arrs)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.ref.lib.ref_system_destroy(self.h)
            self.h = C.c_void_p()

    def build_table(self, list_cutoff, extra_pad=0, vec=True) -> Table:
        total = C.c_size_t()
        self.ref._check(self.ref.lib.ref_table_build(self.h, list_cutoff, extra_pad, int(vec),
                                                     C.byref(total)))
        return self.export_table(list_cutoff, total.value)

    def export_table(self, cutoff, total) -> Table:
        n = self.n
        nn, n8, n16 = (np.zeros(n, np.uint32) for _ in range(3))
        off = np.zeros(n, np.uint64)
        idx = np.zeros(total, np.int32)
        sc = np.zeros(total)
        self.ref._check(self.ref.lib.ref_table_export(self.h, _ptr(nn, _up), _ptr(n8, _up),
                                                      _ptr(n16, _up), _ptr(off, _lp),
                                                      _ptr(idx, _ip), _ptr(sc)))
        return Table(cutoff, nn, n8, n16, off, idx, sc)

    def set_table(self, t: Table):
        self.ref._check(self.ref.lib.ref_table_set(
            self.h, t.cutoff, _ptr(np.ascontiguousarray(t.nnvlst), _up),
            _ptr(np.ascontiguousarray(t.nvloop8), _up), _ptr(np.ascontiguousarray(t.nvloop16), _up),
            _ptr(np.ascontiguousarray(t.offset), _lp), _ptr(np.ascontiguousarray(t.indices), _ip),
            int(t.indices.shape[0])))

    def brute_force_pairs(self, cutoff) -> np.ndarray:
        cap = 1 << 20
        out = np.zeros(2 * cap, np.int32)
        npairs = C.c_size_t()
        self.ref._check(self.ref.lib.ref_brute_force_pairs(self.h, cutoff, _ptr(out, _ip), cap,
                                                           C.byref(npairs)))
        return out[: 2 * npairs.value].reshape(-1, 2).astype(np.int64)

    def forces(self, kind: str, cutoff, p1=0.0, p2=0.0, shift=False, vec=True):
        k = {"lj": 0, "ewald_real": 1, "halgren": 2}[kind]
        f = [np.zeros(self.n) for _ in range(3)]
        e = C.c_double()
        self.ref._check(self.ref.lib.ref_forces(self.h, k, int(vec), cutoff, p1, p2, int(shift),
                                                *(_ptr(v) for v in f), C.byref(e)))
        return np.stack(f, 1), e.value

    def field(self, kind: str, cutoff, thole_a, mu=None, vec=True):
        n = self.n
        if mu is None:
            mu = np.zeros((n, 3))
        m = [np.ascontiguousarray(mu[:, a]) for a in range(3)]
        e = [np.zeros(n) for _ in range(3)]
        self.ref._check(self.ref.lib.ref_field(self.h, 0 if kind == "tmatxb" else 1, int(vec),
                                               cutoff, thole_a, *(_ptr(v) for v in m),
                                               *(_ptr(v) for v in e)))
        return np.stack(e, 1)

    def jacobi(self, cutoff, thole_a, tol, max_iter):
        m = [np.zeros(self.n) for _ in range(3)]
        res = C.c_double()
        rc = self.ref.lib.ref_jacobi(self.h, cutoff, thole_a, tol, max_iter,
                                     *(_ptr(v) for v in m), C.byref(res))
        if rc == 4:
            err = OracleError(rc, self.ref.lib.ref_last_error().decode())
            err.last_residual = res.value
            raise err
        self.ref._check(rc)
        return np.stack(m, 1)


# ------------------------------------------------------------ CPU-baseline port
def fast_port_path() -> str:
    isa = ref_isa()
    p = os.path.join(HERE, f"libmdo_fast_{isa}.so")
    if not os.path.exists(p) or os.path.getmtime(p) < os.path.getmtime(os.path.join(HERE, "mdo_fast.c")):
        subprocess.check_call(["make", "-s", "-C", HERE, "fast"])
    return p


class FastPort:
    """mdo_fast.c: closed-form half-list CPU kernels (the CPU baseline's port leg)."""

    def __init__(self, path: str | None = None):
        self.lib = C.CDLL(path or fast_port_path())
        L = self.lib
        L.mdf_mpole.argtypes = [C.POINTER(MdoSystem), C.POINTER(MdoTable), C.c_double, C.c_double,
                                C.c_double, C.c_int, _dp, _dp, _dp, _dp]
        self.last_virial = None
        L.mdf_perm_field.argtypes = [C.POINTER(MdoSystem), C.POINTER(MdoTable), C.c_double,
                                     C.c_double, C.c_double, C.c_int, _dp]
        L.mdf_tmatvec.argtypes = [C.POINTER(MdoSystem), C.POINTER(MdoTable), C.c_double,
                                  C.c_double, C.c_double, _dp, _dp]

    def mpole(self, s, t, alpha, cutoff, electric=1.0, exclude=True, st=None, tt=None):
        st = st or s.as_struct()
        tt = tt or t.as_struct()
        f = np.zeros((s.n, 3))
        tq = np.zeros((s.n, 3))
        e = C.c_double()
        w = np.zeros(9)
        self.lib.mdf_mpole(C.byref(st), C.byref(tt), alpha, cutoff, electric, int(exclude),
                           _ptr(f), _ptr(tq), C.byref(e), _ptr(w))
        self.last_virial = w.reshape(3, 3)  # pair virial sum d_a F_b (F on i)
        return f, tq, e.value

    def perm_field(self, s, t, alpha, cutoff, thole_a, exclude=True, st=None, tt=None):
        st = st or s.as_struct()
        tt = tt or t.as_struct()
        e = np.zeros((s.n, 3))
        self.lib.mdf_perm_field(C.byref(st), C.byref(tt), alpha, cutoff, thole_a, int(exclude),
                                _ptr(e))
        return e

    def tmatvec(self, s, t, alpha, cutoff, thole_a, mu, st=None, tt=None):
        st = st or s.as_struct()
        tt = tt or t.as_struct()
        mu = np.ascontiguousarray(mu, np.float64)
        e = np.zeros((s.n, 3))
        self.lib.mdf_tmatvec(C.byref(st), C.byref(tt), alpha, cutoff, thole_a, _ptr(mu), _ptr(e))
        return e
