// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library (/root/reference/proj,
// compiled from its own sources by oracle/Makefile into oracle/_ref/). It lets
// the Python tests and bench.py's reference arm call the reference's scalar
// ("Rel") and vectorised ("Vec") kernels on plain arrays. Nothing here is
// product code; no reference source is copied into this repository.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "mdvec/kernels.hpp"
#include "mdvec/neighbors.hpp"
#include "mdvec/polar.hpp"
#include "mdvec/system.hpp"

using namespace mdvec;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ContractViolation& e) {
    g_err = e.what();
    return 1;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return 2;
  } catch (const SingularityError& e) {
    g_err = e.what();
    return 3;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

struct RefSystem {
  ParticleSystem sys;
  std::unique_ptr<NeighborTable> table;
  LaneConfig lanes;
  PairWorkspace ws;
};

void fill(PaddedRealArray& a, const double* src, std::size_t n) {
  a = PaddedRealArray(n);
  std::memcpy(a.data(), src, n * sizeof(double));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Builds a ParticleSystem from SoA arrays (proj/include/mdvec/system.hpp:12-25).
int ref_system_create(void** out, std::size_t n, double lx, double ly, double lz,
                      const double* x, const double* y, const double* z, const double* q,
                      const double* sig, const double* eps, const double* r0,
                      const double* heps, const double* pol) {
  return guard([&] {
    auto* r = new RefSystem();
    r->sys.box = {lx, ly, lz};
    r->sys.n_sites = n;
    fill(r->sys.x, x, n);
    fill(r->sys.y, y, n);
    fill(r->sys.z, z, n);
    fill(r->sys.charge, q, n);
    fill(r->sys.lj_sigma, sig, n);
    fill(r->sys.lj_epsilon, eps, n);
    fill(r->sys.hal_r0, r0, n);
    fill(r->sys.hal_epsilon, heps, n);
    fill(r->sys.polarizability, pol, n);
    *out = r;
  });
}

void ref_system_destroy(void* h) { delete static_cast<RefSystem*>(h); }

// proj/src/system.cpp:65-173 (generator) -> arrays
int ref_generate_system(int kind, std::size_t n, double lx, double ly, double lz,
                        std::uint64_t seed, double min_sep, double* x, double* y, double* z,
                        double* q, double* sig, double* eps, double* r0, double* heps,
                        double* pol) {
  return guard([&] {
    ParticleSystem s = generate_system(
        kind == 0 ? SystemKind::kLatticeWaterLike : SystemKind::kUniformRandom, n,
        {lx, ly, lz}, seed, min_sep);
    std::memcpy(x, s.x.data(), n * 8);
    std::memcpy(y, s.y.data(), n * 8);
    std::memcpy(z, s.z.data(), n * 8);
    std::memcpy(q, s.charge.data(), n * 8);
    std::memcpy(sig, s.lj_sigma.data(), n * 8);
    std::memcpy(eps, s.lj_epsilon.data(), n * 8);
    std::memcpy(r0, s.hal_r0.data(), n * 8);
    std::memcpy(heps, s.hal_epsilon.data(), n * 8);
    std::memcpy(pol, s.polarizability.data(), n * 8);
  });
}

void ref_random_dipoles(std::size_t n, std::uint64_t seed, double mag, double* mx, double* my,
                        double* mz) {
  ParticleSystem s;
  s.n_sites = n;
  PolarizationState st = random_dipoles(s, seed, mag);
  std::memcpy(mx, st.mu_x.data(), n * 8);
  std::memcpy(my, st.mu_y.data(), n * 8);
  std::memcpy(mz, st.mu_z.data(), n * 8);
}

// proj/src/neighbors.cpp:10-36 + neighbors_vec.cpp:8-94 (vec=1) or
// neighbors_ref.cpp:8-52 (vec=0). Total padded slots -> *total.
int ref_table_build(void* h, double list_cutoff, std::size_t extra_pad, int vec,
                    std::size_t* total) {
  auto* r = static_cast<RefSystem*>(h);
  return guard([&] {
    CellGrid g = build_cell_grid(r->sys, list_cutoff);
    r->table = std::make_unique<NeighborTable>(
        vec ? build_neighbor_table(r->sys, g, list_cutoff, extra_pad)
            : build_neighbor_table_reference(r->sys, g, list_cutoff));
    *total = r->table->indices.logical_len();
  });
}

// Replaces the system's table with a caller-supplied one (reference layout).
int ref_table_set(void* h, double cutoff, const std::uint32_t* nnvlst, const std::uint32_t* nv8,
                  const std::uint32_t* nv16, const std::uint64_t* offset,
                  const std::int32_t* indices, std::size_t total) {
  auto* r = static_cast<RefSystem*>(h);
  return guard([&] {
    auto t = std::make_unique<NeighborTable>();
    const std::size_t n = r->sys.n_sites;
    t->cutoff = cutoff;
    t->n_sites = n;
    t->nnvlst.assign(nnvlst, nnvlst + n);
    t->nvloop8.assign(nv8, nv8 + n);
    t->nvloop16.assign(nv16, nv16 + n);
    t->offset.assign(offset, offset + n);
    t->indices = PaddedIndexArray(total);
    t->scale = PaddedRealArray(total);
    std::memcpy(t->indices.data(), indices, total * 4);
    for (std::size_t i = 0; i < n; ++i)
      for (std::uint32_t k = 0; k < t->nvloop16[i]; ++k)
        t->scale[t->offset[i] + k] = k < t->nnvlst[i] ? 1.0 : 0.0;
    r->table = std::move(t);
  });
}

int ref_table_export(void* h, std::uint32_t* nnvlst, std::uint32_t* nv8, std::uint32_t* nv16,
                     std::uint64_t* offset, std::int32_t* indices, double* scale) {
  auto* r = static_cast<RefSystem*>(h);
  return guard([&] {
    const NeighborTable& t = *r->table;
    for (std::size_t i = 0; i < t.n_sites; ++i) {
      nnvlst[i] = t.nnvlst[i];
      nv8[i] = t.nvloop8[i];
      nv16[i] = t.nvloop16[i];
      offset[i] = t.offset[i];
    }
    std::memcpy(indices, t.indices.data(), t.indices.logical_len() * 4);
    std::memcpy(scale, t.scale.data(), t.scale.logical_len() * 8);
  });
}

int ref_brute_force_pairs(void* h, double cutoff, std::int32_t* out, std::size_t cap,
                          std::size_t* npairs) {
  auto* r = static_cast<RefSystem*>(h);
  return guard([&] {
    auto p = brute_force_pairs(r->sys, cutoff);
    *npairs = p.size();
    for (std::size_t k = 0; k < p.size() && k < cap; ++k) {
      out[2 * k] = p[k].first;
      out[2 * k + 1] = p[k].second;
    }
  });
}

// kind: 0 lj, 1 ewald_real, 2 halgren. vec selects the Vec path.
int ref_forces(void* h, int kind, int vec, double cutoff, double p1, double p2, int shift,
               double* fx, double* fy, double* fz, double* energy) {
  auto* r = static_cast<RefSystem*>(h);
  return guard([&] {
    const std::size_t n = r->sys.n_sites;
    ForceAccumulator out(n);
    if (kind == 0) {
      LjParams p{cutoff, shift != 0};
      vec ? lj_forces_vectorized(r->sys, *r->table, p, r->lanes, r->ws, out)
          : lj_forces_scalar(r->sys, *r->table, p, out);
    } else if (kind == 1) {
      EwaldRealParams p{p1, cutoff};
      vec ? ewald_real_forces_vectorized(r->sys, *r->table, p, r->lanes, r->ws, out)
          : ewald_real_forces_scalar(r->sys, *r->table, p, out);
    } else {
      HalgrenParams p{cutoff, p1, p2};
      vec ? halgren_forces_vectorized(r->sys, *r->table, p, r->lanes, r->ws, out)
          : halgren_forces_scalar(r->sys, *r->table, p, out);
    }
    std::memcpy(fx, out.fx.data(), n * 8);
    std::memcpy(fy, out.fy.data(), n * 8);
    std::memcpy(fz, out.fz.data(), n * 8);
    *energy = out.energy;
  });
}

// kind: 0 dipole_field_matvec (mu given), 1 permanent_field.
int ref_field(void* h, int kind, int vec, double cutoff, double thole_a, const double* mx,
              const double* my, const double* mz, double* ex, double* ey, double* ez) {
  auto* r = static_cast<RefSystem*>(h);
  return guard([&] {
    const std::size_t n = r->sys.n_sites;
    FieldArrays out(n);
    PolarParams p{cutoff, thole_a};
    if (kind == 0) {
      PolarizationState st;
      fill(st.mu_x, mx, n);
      fill(st.mu_y, my, n);
      fill(st.mu_z, mz, n);
      st.thole_a = thole_a;
      vec ? dipole_field_matvec_vectorized(r->sys, *r->table, st, p, r->lanes, r->ws, out)
          : dipole_field_matvec_scalar(r->sys, *r->table, st, p, out);
    } else {
      vec ? permanent_field_vectorized(r->sys, *r->table, p, r->lanes, r->ws, out)
          : permanent_field_scalar(r->sys, *r->table, p, out);
    }
    std::memcpy(ex, out.ex.data(), n * 8);
    std::memcpy(ey, out.ey.data(), n * 8);
    std::memcpy(ez, out.ez.data(), n * 8);
  });
}

// proj/src/polar_scalar.cpp:161-198
int ref_jacobi(void* h, double cutoff, double thole_a, double tol, std::size_t max_iter,
               double* mx, double* my, double* mz, double* last_residual) {
  auto* r = static_cast<RefSystem*>(h);
  try {
    PolarParams p{cutoff, thole_a};
    PolarizationState st = jacobi_polarization_solve(r->sys, *r->table, p, tol, max_iter);
    const std::size_t n = r->sys.n_sites;
    std::memcpy(mx, st.mu_x.data(), n * 8);
    std::memcpy(my, st.mu_y.data(), n * 8);
    std::memcpy(mz, st.mu_z.data(), n * 8);
    return 0;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    *last_residual = e.last_residual;
    return 4;
  } catch (const ContractViolation& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

}  // extern "C"
