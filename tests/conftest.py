"""Shared fixtures. `-m gpu` tests need a B200 and call the product through the
C ABI (libmdg.so); everything else runs on CPU against the oracle (oracle/)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    # the parity tests run on small systems: let them take the buffered-row
    # path (nlist.cu kernel_rows) that production sizes (>= 50k sites) take;
    # tests switch MDG_PRUNE_BUFFER=0 where they need the plain rows
    os.environ.setdefault("MDG_PRUNE_MIN_SITES", "0")
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref), when built here."""
    from oracle.oracle import RefLib, ref_library_path
    if ref_library_path() is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return RefLib()


@pytest.fixture(scope="session")
def mdg():
    import paper_1906_01211_b200 as m
    m.load_library()
    return m


@pytest.fixture(scope="session")
def engine(mdg):
    """One GPU context for the session (capacity covers the config-1/2 box)."""
    import torch  # noqa: F401  (device visibility only)
    e = mdg.Engine(n_capacity=200_000)
    yield e
    e.close()


def to_oracle_system(s):
    """ParticleSystem (product) -> oracle.System (same arrays, no copy semantics)."""
    from oracle.oracle import System
    return System(tuple(s.box), np.asarray(s.x), np.asarray(s.y), np.asarray(s.z),
                  np.asarray(s.charge), np.asarray(s.lj_sigma), np.asarray(s.lj_epsilon),
                  np.asarray(s.hal_r0), np.asarray(s.hal_epsilon), np.asarray(s.polarizability),
                  molecule=getattr(s, "molecule", None), dipole=getattr(s, "dipole", None),
                  quadrupole=getattr(s, "quadrupole", None))


def rel(a, b):
    scale = max(abs(a), abs(b))
    return abs(a - b) / scale if scale > 0 else 0.0


def force_err_rms(f, g):
    """max |f - g| per component / RMS force of g (BASELINE: 1e-8 x RMS)."""
    f, g = np.asarray(f), np.asarray(g)
    rms = np.sqrt(np.mean(g * g)) + 1e-300
    return float(np.max(np.abs(f - g)) / rms)


def force_err_max(f, g):
    """reference bench metric: max |f - g| / max |g| (proj/src/bench.cpp:32-45)."""
    f, g = np.asarray(f), np.asarray(g)
    return float(np.max(np.abs(f - g)) / (np.max(np.abs(g)) + 1e-300))
