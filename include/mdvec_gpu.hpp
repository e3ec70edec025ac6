// mdvec_gpu.hpp -- C++ drop-in over the C ABI (mdg.h) with the reference's
// own types, signatures and exception taxonomy.
//
// A maintainer of the reference library (`mdvec`, proj/include/mdvec/*.hpp)
// includes this header next to the reference headers and links libmdg.so.
// Every function mirrors a reference entry point and keeps its semantics:
// OVERWRITE the output (`out.reset()` first, proj/src/kernels_scalar.cpp:13),
// validate like proj/src/kernels_impl.hpp:8-20, throw ContractViolation /
// CapacityError / SingularityError / ConvergenceError
// (proj/include/mdvec/common.hpp:12-32). The pair set is exactly the
// NeighborTable passed in (mdg_nlist_import), so results match the reference
// kernels on the same table within the tolerances in DESIGN.md.
//
//   reference                                   drop-in
//   build_cell_grid + build_neighbor_table      mdvec::gpu::build_neighbor_table
//   lj_forces_{scalar,vectorized}               mdvec::gpu::lj_forces
//   ewald_real_forces_*                         mdvec::gpu::ewald_real_forces
//   halgren_forces_*                            mdvec::gpu::halgren_forces
//   dipole_field_matvec_*                       mdvec::gpu::dipole_field_matvec
//   permanent_field_*                           mdvec::gpu::permanent_field
//   jacobi_polarization_solve                   mdvec::gpu::jacobi_polarization_solve
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "mdg.h"
#include "mdvec/kernels.hpp"
#include "mdvec/neighbors.hpp"
#include "mdvec/polar.hpp"

namespace mdvec::gpu {

inline void check(int rc, double residual = 0.0) {
  if (rc == MDG_OK) return;
  const std::string msg = mdg_last_error();
  switch (rc) {
    case MDG_CONTRACT: throw ContractViolation(msg);
    case MDG_CAPACITY: throw CapacityError(msg);
    case MDG_SINGULARITY: throw SingularityError(msg);
    case MDG_CONVERGENCE: throw ConvergenceError(msg, residual);
    default: throw std::runtime_error("mdg: " + msg);
  }
}

// One device context (one GPU, one stream, capacity fixed up front: the
// reference's preallocation contract, proj/tests/test_layout.cpp:215-237).
class Engine {
 public:
  explicit Engine(std::size_t n_capacity, int device = 0) {
    check(mdg_ctx_create(&ctx_, device, static_cast<int64_t>(n_capacity), 0));
  }
  ~Engine() { mdg_ctx_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  mdg_ctx* get() const { return ctx_; }

  // Uploads the ParticleSystem when it is not the one already resident.
  void bind(const ParticleSystem& s) {
    if (bound_ == &s && bound_n_ == s.n_sites) return;
    check(mdg_system_upload(ctx_, static_cast<int64_t>(s.n_sites), s.box.lx, s.box.ly,
                            s.box.lz, s.x.data(), s.y.data(), s.z.data(), s.charge.data(),
                            s.lj_sigma.data(), s.lj_epsilon.data(), s.hal_r0.data(),
                            s.hal_epsilon.data(), s.polarizability.data()));
    bound_ = &s;
    bound_n_ = s.n_sites;
    table_ = nullptr;
  }

  // Feeds the caller's table (slot 2) so the kernel sees exactly its pairs.
  void bind(const ParticleSystem& s, const NeighborTable& t) {
    bind(s);
    if (table_ == &t) return;
    std::vector<std::uint64_t> off(t.offset.begin(), t.offset.end());
    check(mdg_nlist_import(ctx_, kTableSlot, t.cutoff, MDG_SITES_ATOMIC, t.nnvlst.data(),
                           off.data(), t.indices.data()));
    table_ = &t;
  }

  static constexpr int kTableSlot = 2;

 private:
  mdg_ctx* ctx_ = nullptr;
  const ParticleSystem* bound_ = nullptr;
  std::size_t bound_n_ = 0;
  const NeighborTable* table_ = nullptr;
};

// build_neighbor_table (proj/include/mdvec/neighbors.hpp:48-50): built on the
// device, returned in the reference layout (segments ascending in j).
inline NeighborTable build_neighbor_table(Engine& e, const ParticleSystem& s,
                                          double list_cutoff) {
  e.bind(s);
  check(mdg_nlist_build(e.get(), 0, list_cutoff, MDG_SITES_ATOMIC));
  int64_t half = 0, padded = 0;
  check(mdg_nlist_size(e.get(), 0, &half, &padded));
  const std::size_t n = s.n_sites;
  NeighborTable t;
  t.cutoff = list_cutoff;
  t.n_sites = n;
  t.nnvlst.resize(n);
  t.nvloop8.resize(n);
  t.nvloop16.resize(n);
  std::vector<std::uint64_t> off(n);
  t.indices = PaddedIndexArray(static_cast<std::size_t>(padded));
  check(mdg_nlist_export(e.get(), 0, t.nnvlst.data(), t.nvloop8.data(), t.nvloop16.data(),
                         off.data(), t.indices.data(), padded));
  t.offset.assign(off.begin(), off.end());
  t.scale = PaddedRealArray(static_cast<std::size_t>(padded));
  for (std::size_t i = 0; i < n; ++i)
    for (std::uint32_t k = 0; k < t.nvloop16[i]; ++k)
      t.scale[t.offset[i] + k] = k < t.nnvlst[i] ? 1.0 : 0.0;
  return t;
}

inline void lj_forces(Engine& e, const ParticleSystem& s, const NeighborTable& t,
                      const LjParams& p, ForceAccumulator& out) {
  e.bind(s, t);
  out.reset();
  check(mdg_lj_forces(e.get(), Engine::kTableSlot, p.cutoff, p.shift ? 1 : 0, 0, out.fx.data(),
                      out.fy.data(), out.fz.data(), &out.energy, nullptr));
}

inline void ewald_real_forces(Engine& e, const ParticleSystem& s, const NeighborTable& t,
                              const EwaldRealParams& p, ForceAccumulator& out) {
  e.bind(s, t);
  out.reset();
  check(mdg_ewald_real_forces(e.get(), Engine::kTableSlot, p.alpha, p.cutoff, 1.0, 0,
                              out.fx.data(), out.fy.data(), out.fz.data(), &out.energy,
                              nullptr));
}

inline void halgren_forces(Engine& e, const ParticleSystem& s, const NeighborTable& t,
                           const HalgrenParams& p, ForceAccumulator& out) {
  e.bind(s, t);
  out.reset();
  check(mdg_halgren_forces(e.get(), Engine::kTableSlot, p.cutoff, p.delta, p.gamma, 0,
                           out.fx.data(), out.fy.data(), out.fz.data(), &out.energy, nullptr));
}

inline void dipole_field_matvec(Engine& e, const ParticleSystem& s, const NeighborTable& t,
                                const PolarizationState& st, const PolarParams& p,
                                FieldArrays& out) {
  e.bind(s, t);
  out.reset();
  // the reference mat-vec reads state.thole_a (proj/src/polar_scalar.cpp:79)
  check(mdg_tmatvec(e.get(), Engine::kTableSlot, 0.0, p.cutoff, st.thole_a, st.mu_x.data(),
                    st.mu_y.data(), st.mu_z.data(), out.ex.data(), out.ey.data(),
                    out.ez.data()));
}

inline void permanent_field(Engine& e, const ParticleSystem& s, const NeighborTable& t,
                            const PolarParams& p, FieldArrays& out) {
  e.bind(s, t);
  out.reset();
  check(mdg_perm_field(e.get(), Engine::kTableSlot, 0.0, p.cutoff, p.thole_a, 0, out.ex.data(),
                       out.ey.data(), out.ez.data()));
}

inline PolarizationState jacobi_polarization_solve(Engine& e, const ParticleSystem& s,
                                                   const NeighborTable& t,
                                                   const PolarParams& p, double tol,
                                                   std::size_t max_iter) {
  e.bind(s, t);
  PolarizationState mu;
  mu.thole_a = p.thole_a;
  mu.mu_x = PaddedRealArray(s.n_sites);
  mu.mu_y = PaddedRealArray(s.n_sites);
  mu.mu_z = PaddedRealArray(s.n_sites);
  int64_t iters = 0;
  double resid = 0.0;
  const int rc = mdg_polar_solve_jacobi(e.get(), Engine::kTableSlot, p.cutoff, p.thole_a, tol,
                                        static_cast<int64_t>(max_iter), mu.mu_x.data(),
                                        mu.mu_y.data(), mu.mu_z.data(), &iters, &resid);
  check(rc, resid);
  return mu;
}

}  // namespace mdvec::gpu
