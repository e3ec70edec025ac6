// wrapper_check.cpp -- TEST INFRASTRUCTURE: the C++ drop-in (include/mdvec_gpu.hpp)
// used with the reference's own types, side by side with the reference's own
// kernels (oracle/_ref objects), on the reference's own random systems. Built
// here by `make -C oracle wrapper` (needs /root/reference headers), run on the
// GPU box by tests/test_gpu_wrapper.py. Exit code 0 = every check passed.
#include <cmath>
#include <cstdio>
#include <string>

#include "mdvec_gpu.hpp"

using namespace mdvec;

static int g_fail = 0;

static void expect(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "[PASS]" : "[FAIL]", what.c_str());
  if (!ok) ++g_fail;
}

static double max_rel(const ForceAccumulator& a, const ForceAccumulator& b, std::size_t n) {
  double scale = 1e-300, worst = 0;
  for (std::size_t i = 0; i < n; ++i)
    scale = std::fmax(scale, std::fmax(std::fabs(a.fx[i]), std::fmax(std::fabs(a.fy[i]),
                                                                      std::fabs(a.fz[i]))));
  for (std::size_t i = 0; i < n; ++i)
    worst = std::fmax(worst, std::fmax(std::fabs(a.fx[i] - b.fx[i]),
                                       std::fmax(std::fabs(a.fy[i] - b.fy[i]),
                                                 std::fabs(a.fz[i] - b.fz[i]))));
  return worst / scale;
}

static double field_rel(const FieldArrays& a, const FieldArrays& b, std::size_t n) {
  double scale = 1e-300, worst = 0;
  for (std::size_t i = 0; i < n; ++i)
    scale = std::fmax(scale, std::fmax(std::fabs(a.ex[i]), std::fmax(std::fabs(a.ey[i]),
                                                                      std::fabs(a.ez[i]))));
  for (std::size_t i = 0; i < n; ++i)
    worst = std::fmax(worst, std::fmax(std::fabs(a.ex[i] - b.ex[i]),
                                       std::fmax(std::fabs(a.ey[i] - b.ey[i]),
                                                 std::fabs(a.ez[i] - b.ez[i]))));
  return worst / scale;
}

int main() {
  gpu::Engine eng(4096);
  for (std::uint64_t seed = 1; seed <= 4; ++seed) {
    for (std::size_t n : {16u, 100u, 333u, 2000u}) {
      const double L = n == 2000 ? 27.0 : 12.0;
      ParticleSystem s = generate_system(SystemKind::kUniformRandom, n, {L, L, L}, seed);
      CellGrid g = build_cell_grid(s, 3.7);
      NeighborTable t = build_neighbor_table(s, g, 3.7);
      const std::string tag = " seed " + std::to_string(seed) + " n " + std::to_string(n);

      NeighborTable tg = gpu::build_neighbor_table(eng, s, 3.7);
      expect(table_pairs(tg) == table_pairs(t), "pair set == reference" + tag);

      ForceAccumulator a(n), b(n);
      lj_forces_scalar(s, t, {3.0, false}, a);
      gpu::lj_forces(eng, s, t, {3.0, false}, b);
      expect(std::fabs(a.energy - b.energy) <= 1e-9 * std::fabs(a.energy) &&
                 max_rel(a, b, n) <= 1e-9,
             "lj" + tag);
      ewald_real_forces_scalar(s, t, {0.4, 3.7}, a);
      gpu::ewald_real_forces(eng, s, t, {0.4, 3.7}, b);
      expect(std::fabs(a.energy - b.energy) <= 1e-9 * std::fabs(a.energy) &&
                 max_rel(a, b, n) <= 1e-9,
             "ewald_real" + tag);
      halgren_forces_scalar(s, t, {3.0}, a);
      gpu::halgren_forces(eng, s, t, {3.0}, b);
      expect(std::fabs(a.energy - b.energy) <= 1e-9 * std::fabs(a.energy) &&
                 max_rel(a, b, n) <= 1e-9,
             "halgren" + tag);
      PolarizationState st = random_dipoles(s, seed + 100);
      FieldArrays fa(n), fb(n);
      dipole_field_matvec_scalar(s, t, st, {3.0, 0.39}, fa);
      gpu::dipole_field_matvec(eng, s, t, st, {3.0, 0.39}, fb);
      expect(field_rel(fa, fb, n) <= 1e-9, "tmatxb" + tag);
      permanent_field_scalar(s, t, {3.0, 0.39}, fa);
      gpu::permanent_field(eng, s, t, {3.0, 0.39}, fb);
      expect(field_rel(fa, fb, n) <= 1e-9, "perm_field" + tag);
    }
  }
  // error taxonomy: kernel cutoff beyond the list, non-convergence
  {
    ParticleSystem s = generate_system(SystemKind::kUniformRandom, 30, {9, 9, 9}, 13);
    NeighborTable t = build_neighbor_table(s, build_cell_grid(s, 3.0), 3.0);
    ForceAccumulator out(30);
    bool threw = false;
    try {
      gpu::lj_forces(eng, s, t, {3.5, false}, out);
    } catch (const ContractViolation&) {
      threw = true;
    }
    expect(threw, "ContractViolation for cutoff > list cutoff");
    threw = false;
    try {
      gpu::jacobi_polarization_solve(eng, s, t, {3.0, 0.39}, 1e-300, 2);
    } catch (const ConvergenceError& e) {
      threw = e.last_residual > 0;
    }
    expect(threw, "ConvergenceError with last_residual");
    PolarizationState ref = jacobi_polarization_solve(
        generate_system(SystemKind::kUniformRandom, 15, {9, 9, 9}, 21),
        build_neighbor_table(generate_system(SystemKind::kUniformRandom, 15, {9, 9, 9}, 21),
                             build_cell_grid(generate_system(SystemKind::kUniformRandom, 15,
                                                             {9, 9, 9}, 21),
                                             3.0),
                             3.0),
        {3.0, 0.39}, 1e-12, 500);
    ParticleSystem s15 = generate_system(SystemKind::kUniformRandom, 15, {9, 9, 9}, 21);
    NeighborTable t15 = build_neighbor_table(s15, build_cell_grid(s15, 3.0), 3.0);
    PolarizationState got = gpu::jacobi_polarization_solve(eng, s15, t15, {3.0, 0.39}, 1e-12, 500);
    double worst = 0;
    for (std::size_t i = 0; i < 15; ++i)
      worst = std::fmax(worst, std::fabs(got.mu_x[i] - ref.mu_x[i]) +
                                   std::fabs(got.mu_y[i] - ref.mu_y[i]) +
                                   std::fabs(got.mu_z[i] - ref.mu_z[i]));
    expect(worst <= 1e-10, "jacobi == reference jacobi");
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
