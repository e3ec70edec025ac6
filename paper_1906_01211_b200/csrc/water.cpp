// water.cpp -- synthetic 3-site water fixtures for BASELINE.json configs 0-4
// and the host twin of the device's Halgren site reduction.
//
// The reference generator (proj/src/system.cpp:65-173) places single sites
// with random parameters; BASELINE.json asks for rigid 3-site waters, so this
// generator is new. It follows the reference's lattice rule (m = ceil(cbrt
// n_mol), O at (i + 1/2) spacing + U(+-0.05 spacing)) and seeds
// std::mt19937_64 like the reference (proj/src/system.cpp:84). When m^3 >
// n_mol the occupied lattice slots are a seeded random subset, so there is
// no void slab. All distributions are written out explicitly (no
// implementation-defined std:: distributions), so the fixture is
// reproducible bit-for-bit on any host.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/mdg.h"

namespace {

struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t seed) : g(seed) {}
  double uniform() { return (double)(g() >> 11) * 0x1.0p-53; }  // [0, 1)
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  double normal(double mean, double sd) {  // Box-Muller, one value per call
    double u1 = uniform();
    const double u2 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    return mean + sd * std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

double wrap_into(double p, double L) {
  p -= L * std::floor(p / L);
  if (p >= L) p = 0.0;
  if (p < 0.0) p = 0.0;
  return p;
}

double wrap1(double d, double L) {
  const double t = std::fma(-std::nearbyint(d * (1.0 / L)), L, d);
  return (t >= 0.5 * L) ? t - L : t;
}

// wrap_into with every op separately rounded (device twin: core.cu)
double wrap_into_exact(double p, double L) {
  volatile double k = std::floor(p / L);
  volatile double m = L * k;
  volatile double r = p - m;
  double q = r;
  if (q >= L) q = 0.0;
  if (q < 0.0) q = 0.0;
  return q;
}

}  // namespace

extern "C" {

int mdg_water_generate(int64_t n_mol, double box, uint64_t seed, int model, double* x,
                       double* y, double* z, int32_t* molecule, double* charge,
                       double* lj_sigma, double* lj_epsilon, double* hal_r0,
                       double* hal_epsilon, double* polarizability, int32_t* hred_parent,
                       double* hred_factor, double* dipole, double* quadrupole) {
  if (n_mol < 1 || !(box > 0) || (model != 0 && model != 1)) return MDG_CONTRACT;
  Rng rng(seed);
  int64_t m = 1;
  while (m * m * m < n_mol) ++m;
  const int64_t slots = m * m * m;
  std::vector<int64_t> slot(slots);
  for (int64_t k = 0; k < slots; ++k) slot[k] = k;
  if (slots > n_mol) {
    for (int64_t k = slots - 1; k > 0; --k) {
      const int64_t j = (int64_t)(rng.g() % (uint64_t)(k + 1));
      std::swap(slot[k], slot[j]);
    }
    slot.resize(n_mol);
    std::sort(slot.begin(), slot.end());
  }
  const double sp = box / (double)m;
  const double jit = 0.05 * sp;
  // body frame: O at origin, H in the xz plane, O-H 0.9572 A, H-O-H 104.52 deg
  const double b = 0.9572, half = 0.5 * 104.52 * 3.141592653589793 / 180.0;
  const double hb[2][3] = {{b * std::sin(half), 0.0, b * std::cos(half)},
                           {-b * std::sin(half), 0.0, b * std::cos(half)}};
  for (int64_t w = 0; w < n_mol; ++w) {
    const int64_t s = slot[w];
    const int64_t ix = s / (m * m), iy = (s / m) % m, iz = s % m;
    const double ox = (ix + 0.5) * sp + rng.uniform(-jit, jit);
    const double oy = (iy + 0.5) * sp + rng.uniform(-jit, jit);
    const double oz = (iz + 0.5) * sp + rng.uniform(-jit, jit);
    // uniform random rotation (unit quaternion from three uniforms)
    const double u1 = rng.uniform(), u2 = rng.uniform(), u3 = rng.uniform();
    const double tp = 6.283185307179586;
    const double qa = std::sqrt(1 - u1) * std::sin(tp * u2), qb = std::sqrt(1 - u1) * std::cos(tp * u2),
                 qc = std::sqrt(u1) * std::sin(tp * u3), qd = std::sqrt(u1) * std::cos(tp * u3);
    // rotation matrix of quaternion (qd + qa i + qb j + qc k)
    const double R[3][3] = {
        {1 - 2 * (qb * qb + qc * qc), 2 * (qa * qb - qc * qd), 2 * (qa * qc + qb * qd)},
        {2 * (qa * qb + qc * qd), 1 - 2 * (qa * qa + qc * qc), 2 * (qb * qc - qa * qd)},
        {2 * (qa * qc - qb * qd), 2 * (qb * qc + qa * qd), 1 - 2 * (qa * qa + qb * qb)}};
    const int64_t o = 3 * w;
    x[o] = wrap_into(ox, box);
    y[o] = wrap_into(oy, box);
    z[o] = wrap_into(oz, box);
    for (int h = 0; h < 2; ++h) {
      double d[3];
      for (int a = 0; a < 3; ++a)
        d[a] = R[a][0] * hb[h][0] + R[a][1] * hb[h][1] + R[a][2] * hb[h][2];
      x[o + 1 + h] = wrap_into(ox + d[0], box);
      y[o + 1 + h] = wrap_into(oy + d[1], box);
      z[o + 1 + h] = wrap_into(oz + d[2], box);
    }
    for (int k = 0; k < 3; ++k) {
      const int64_t i = o + k;
      const bool O = (k == 0);
      if (molecule) molecule[i] = (int32_t)w;
      if (model == 0) {
        charge[i] = O ? -0.834 : 0.417;
        lj_sigma[i] = O ? 3.1507 : 0.0;
        lj_epsilon[i] = O ? 0.1521 : 0.0;
        hal_r0[i] = O ? 3.405 : 2.655;
        hal_epsilon[i] = O ? 0.110 : 0.0135;
        if (hred_parent) hred_parent[i] = (int32_t)i;
        if (hred_factor) hred_factor[i] = 1.0;
      } else {
        charge[i] = O ? -0.51966 : 0.25983;
        lj_sigma[i] = 0.0;
        lj_epsilon[i] = 0.0;
        hal_r0[i] = O ? 3.405 : 2.655;
        hal_epsilon[i] = O ? 0.110 : 0.0135;
        if (hred_parent) hred_parent[i] = (int32_t)o;
        if (hred_factor) hred_factor[i] = O ? 1.0 : 0.91;
      }
      polarizability[i] = O ? 0.837 : 0.496;
    }
  }
  // permanent dipoles and traceless quadrupoles (second pass: fixed draw order)
  const int64_t n = 3 * n_mol;
  for (int64_t i = 0; i < n; ++i) {
    const double ct = rng.uniform(-1.0, 1.0), ph = 6.283185307179586 * rng.uniform();
    const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
    const double mag = rng.normal(0.15, 0.03);
    double q[6];
    for (int k = 0; k < 6; ++k) q[k] = rng.normal(0.0, 0.1);
    if (model == 0) continue;
    if (dipole) {
      dipole[3 * i] = mag * st * std::cos(ph);
      dipole[3 * i + 1] = mag * st * std::sin(ph);
      dipole[3 * i + 2] = mag * ct;
    }
    if (quadrupole) {
      const double tr = (q[0] + q[3] + q[5]) / 3.0;
      double* Q = quadrupole + 6 * i;
      Q[0] = q[0] - tr;  // xx
      Q[1] = q[1];       // xy
      Q[2] = q[2];       // xz
      Q[3] = q[3] - tr;  // yy
      Q[4] = q[4];       // yz
      Q[5] = q[5] - tr;  // zz
    }
  }
  if (model == 0) {
    if (dipole) std::fill(dipole, dipole + 3 * n, 0.0);
    if (quadrupole) std::fill(quadrupole, quadrupole + 6 * n, 0.0);
  }
  return MDG_OK;
}

int mdg_reduce_sites_host(int64_t n, double lx, double ly, double lz, const double* x,
                          const double* y, const double* z, const int32_t* parent,
                          const double* factor, double* xr, double* yr, double* zr) {
  const double L[3] = {lx, ly, lz};
  const double* P[3] = {x, y, z};
  double* O[3] = {xr, yr, zr};
  for (int64_t i = 0; i < n; ++i) {
    const int64_t p = parent[i];
    if (p < 0 || p >= n) return MDG_CONTRACT;
    for (int a = 0; a < 3; ++a) {
      if (p == i) {
        O[a][i] = P[a][i];
        continue;
      }
      volatile double d = P[a][i] - P[a][p];
      const double w = wrap1(d, L[a]);
      volatile double s = factor[i] * w;
      volatile double t = P[a][p] + s;
      O[a][i] = wrap_into_exact(t, L[a]);
    }
  }
  return MDG_OK;
}

}  // extern "C"
