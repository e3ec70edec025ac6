"""B200-native (sm_100a) FP64 real-space pair engine: a drop-in for the
reference mdvec hot path (neighbour lists, LJ / Ewald / Halgren pair kernels,
Thole/Ewald polarization, real-space multipoles) behind a C ABI."""
from .mdvec import (  # noqa: F401
    CONFIGS, DEBYE, ELECTRIC, SITES_ATOMIC, SITES_VDW, AmoebaParams, CapacityError,
    CharmmParams, ContractViolation, ConvergenceError, CudaError, Engine, EwaldRealParams,
    FieldArrays, ForceAccumulator, HalgrenParams, INTEGRATOR_BAOAB_RESPA, INTEGRATOR_VERLET,
    PREDICT_ASPC, PREDICT_NONE,
    LjParams, MDParams, NeighborTable, ParticleSystem,
    PolarizationState, PolarParams, SingularityError, TERM_MPOLE, TERM_POLAR, TERM_POLAR_FORCE, TERM_VDW,
    dump_system_json, fp64_peak_tflops, host_array, load_library, load_system_json,
    reduce_sites_host,
    water_box)
