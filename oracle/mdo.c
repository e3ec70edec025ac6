/*
 * mdo.c -- CPU ORACLE (test infrastructure only; see mdo.h).
 *
 * Compiled by oracle/Makefile with -O2 -ffp-contract=off so every product
 * and sum is a separately rounded IEEE op; wrap1/dist2 use explicit fma()
 * exactly as proj/include/mdvec/pbc.hpp:27-37 does, so pair selection is
 * bit-identical to the reference and to the device kernels.
 */
#include "mdo.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char* mdo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ PBC */

/* proj/include/mdvec/pbc.hpp:27-31 */
double mdo_wrap1(double d, double box_len, double inv_len, double half_len) {
  double t = fma(-nearbyint(d * inv_len), box_len, d);
  return (t >= half_len) ? t - box_len : t;
}

/* proj/include/mdvec/pbc.hpp:35-37 */
double mdo_dist2(double dx, double dy, double dz) { return fma(dx, dx, fma(dy, dy, dz * dz)); }

typedef struct {
  double lx, ly, lz, ix, iy, iz, hx, hy, hz;
} box_t;

static box_t make_box(double lx, double ly, double lz) {
  box_t b = {lx, ly, lz, 1.0 / lx, 1.0 / ly, 1.0 / lz, 0.5 * lx, 0.5 * ly, 0.5 * lz};
  return b;
}

static int box_ok(double lx, double ly, double lz) {
  return lx > 0 && ly > 0 && lz > 0 && isfinite(lx) && isfinite(ly) && isfinite(lz);
}

/* proj/src/pbc.cpp:5-15 */
int mdo_minimum_image(double* dx, double* dy, double* dz, double lx, double ly, double lz) {
  if (!box_ok(lx, ly, lz)) return fail(MDO_CONTRACT, "box edges must be positive and finite");
  if (!isfinite(*dx) || !isfinite(*dy) || !isfinite(*dz))
    return fail(MDO_CONTRACT, "minimum_image: non-finite displacement");
  *dx = mdo_wrap1(*dx, lx, 1.0 / lx, 0.5 * lx);
  *dy = mdo_wrap1(*dy, ly, 1.0 / ly, 0.5 * ly);
  *dz = mdo_wrap1(*dz, lz, 1.0 / lz, 0.5 * lz);
  return MDO_OK;
}

/* displacement i - j, wrapped; returns r2 */
static inline double pair_d(const mdo_system* s, const box_t* b, size_t i, size_t j,
                            double* dx, double* dy, double* dz) {
  *dx = mdo_wrap1(s->x[i] - s->x[j], b->lx, b->ix, b->hx);
  *dy = mdo_wrap1(s->y[i] - s->y[j], b->ly, b->iy, b->hy);
  *dz = mdo_wrap1(s->z[i] - s->z[j], b->lz, b->iz, b->hz);
  return mdo_dist2(*dx, *dy, *dz);
}

/* ------------------------------------------- reference generator restatement */

/* std::mt19937_64 (the reference generator's engine, proj/src/system.cpp:84) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (g->idx >= 312) {
    int k;
    for (k = 0; k < 312 - 156; ++k) {
      uint64_t y = (g->mt[k] & UM) | (g->mt[k + 1] & LM);
      g->mt[k] = g->mt[k + 156] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
    for (; k < 311; ++k) {
      uint64_t y = (g->mt[k] & UM) | (g->mt[k + 1] & LM);
      g->mt[k] = g->mt[k + 156 - 312] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
    uint64_t y = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* libstdc++ uniform_real_distribution<double> over generate_canonical<double,53>
 * with a 64-bit engine: one draw, u / 2^64, clamped below 1. The reference's
 * system.cpp is compiled with -march=native, where GCC contracts
 * `u*(b-a)+a` into one fma; the restatement does the same. */
static double mt64_uniform(mt64* g, double a, double b) {
  double r = (double)mt64_next(g) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return fma(r, b - a, a);
}

/* proj/src/system.cpp:57-61 (contracted the same way as the reference build) */
static double wrap_into(double p, double L) {
  p = fma(-L, floor(p / L), p);
  if (p >= L) p = 0.0;
  return p;
}

/* Full rows (every j != i within cutoff, ascending j) of the listed sites
 * with the reference predicate (wrap1 + dist2, proj/include/mdvec/pbc.hpp:
 * 27-37): the sampled-row oracle of the config-4 parity tests. Candidates
 * come from a cell grid of edge >= cutoff (the 27 surrounding cells,
 * deduplicated; every site when the grid has < 3 cells per axis), so the
 * predicate alone decides membership. counts[k] = row length of sites[k];
 * idx receives the rows back to back (CAPACITY if the total exceeds cap). */
static int cmp_row_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int mdo_rows_for_sites(const mdo_system* s, double cutoff, const int32_t* sites, size_t ns,
                       int32_t* counts, int32_t* idx, size_t cap) {
  const box_t b = make_box(s->lx, s->ly, s->lz);
  const double c2 = cutoff * cutoff;
  const double L[3] = {s->lx, s->ly, s->lz};
  int nc[3];
  for (int a = 0; a < 3; ++a) {
    nc[a] = (int)floor(L[a] / cutoff);
    if (nc[a] < 3) nc[a] = 1;
  }
  const size_t ncell = (size_t)nc[0] * nc[1] * nc[2];
  size_t* start = (size_t*)calloc(ncell + 1, sizeof(size_t));
  int32_t* cell = (int32_t*)malloc(s->n * sizeof(int32_t));
  int32_t* bucket = (int32_t*)malloc(s->n * sizeof(int32_t));
  const double* P[3] = {s->x, s->y, s->z};
  for (size_t j = 0; j < s->n; ++j) {
    int c[3];
    for (int a = 0; a < 3; ++a) {
      c[a] = (int)(P[a][j] / L[a] * nc[a]);
      if (c[a] >= nc[a]) c[a] = nc[a] - 1;
      if (c[a] < 0) c[a] = 0;
    }
    cell[j] = (c[0] * nc[1] + c[1]) * nc[2] + c[2];
    start[cell[j] + 1]++;
  }
  for (size_t k = 0; k < ncell; ++k) start[k + 1] += start[k];
  {
    size_t* fill = (size_t*)malloc(ncell * sizeof(size_t));
    memcpy(fill, start, ncell * sizeof(size_t));
    for (size_t j = 0; j < s->n; ++j) bucket[fill[cell[j]]++] = (int32_t)j;
    free(fill);
  }
  size_t pos = 0;
  int rc = 0;
  for (size_t k = 0; k < ns && rc == 0; ++k) {
    const size_t i = (size_t)sites[k];
    if (i >= s->n) { rc = fail(1, "rows_for_sites: site out of range"); break; }
    const int ci[3] = {cell[i] / (nc[1] * nc[2]), (cell[i] / nc[2]) % nc[1], cell[i] % nc[2]};
    int32_t seen[27];
    int nseen = 0;
    const size_t row0 = pos;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int cc[3] = {((ci[0] + dx) % nc[0] + nc[0]) % nc[0],
                             ((ci[1] + dy) % nc[1] + nc[1]) % nc[1],
                             ((ci[2] + dz) % nc[2] + nc[2]) % nc[2]};
          const int32_t id = (cc[0] * nc[1] + cc[1]) * nc[2] + cc[2];
          int dup = 0;
          for (int q = 0; q < nseen; ++q) dup |= seen[q] == id;
          if (dup) continue;
          seen[nseen++] = id;
          for (size_t t = start[id]; t < start[id + 1]; ++t) {
            const size_t j = (size_t)bucket[t];
            if (j == i) continue;
            double ddx, ddy, ddz;
            if (pair_d(s, &b, i, j, &ddx, &ddy, &ddz) <= c2) {
              if (pos >= cap) { rc = fail(2, "rows_for_sites: capacity"); break; }
              idx[pos++] = (int32_t)j;
            }
          }
        }
    qsort(idx + row0, pos - row0, sizeof(int32_t), cmp_row_i32);
    counts[k] = (int32_t)(pos - row0);
  }
  free(start);
  free(cell);
  free(bucket);
  return rc;
}

/* ------------------------------------------- BASELINE.json water fixtures */
/* Restatement of the BASELINE.json generator rules (reference
 * lattice rule proj/src/system.cpp:87-104, seeded vacant slots, uniform
 * random orientation, O-H 0.9572 A, H-O-H 104.52 deg, the per-config
 * parameters) with explicitly written distributions, so the CPU arm builds
 * its fixture without the product library. tests/test_oracle.py checks it
 * bit-for-bit against mdg_water_generate. */
static double wf_uniform(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
static double wf_uniform_ab(mt64* g, double a, double b) { return a + (b - a) * wf_uniform(g); }
static double wf_normal(mt64* g, double mean, double sd) {
  double u1 = wf_uniform(g);
  const double u2 = wf_uniform(g);
  if (u1 < 1e-300) u1 = 1e-300;
  return mean + sd * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static double wf_wrap(double p, double L) {
  p -= L * floor(p / L);
  if (p >= L) p = 0.0;
  if (p < 0.0) p = 0.0;
  return p;
}
static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int mdo_water_generate(int64_t n_mol, double box, uint64_t seed, int model, double* x,
                       double* y, double* z, int32_t* molecule, double* charge,
                       double* lj_sigma, double* lj_epsilon, double* hal_r0,
                       double* hal_epsilon, double* polarizability, int32_t* hred_parent,
                       double* hred_factor, double* dipole, double* quadrupole) {
  if (n_mol < 1 || !(box > 0) || (model != 0 && model != 1)) return 1;
  mt64* g = (mt64*)malloc(sizeof(mt64));
  mt64_seed(g, seed);
  int64_t m = 1;
  while (m * m * m < n_mol) ++m;
  const int64_t slots = m * m * m;
  int64_t* slot = (int64_t*)malloc((size_t)slots * sizeof(int64_t));
  for (int64_t k = 0; k < slots; ++k) slot[k] = k;
  if (slots > n_mol) { /* Fisher-Yates on the lattice slots, keep the first n_mol */
    for (int64_t k = slots - 1; k > 0; --k) {
      const int64_t j = (int64_t)(mt64_next(g) % (uint64_t)(k + 1));
      const int64_t t = slot[k]; slot[k] = slot[j]; slot[j] = t;
    }
    qsort(slot, (size_t)n_mol, sizeof(int64_t), cmp_i64);
  }
  const double sp = box / (double)m, jit = 0.05 * sp;
  const double bl = 0.9572, half = 0.5 * 104.52 * 3.141592653589793 / 180.0;
  const double hb[2][3] = {{bl * sin(half), 0.0, bl * cos(half)},
                           {-bl * sin(half), 0.0, bl * cos(half)}};
  for (int64_t w = 0; w < n_mol; ++w) {
    const int64_t sl = slot[w];
    const int64_t ix = sl / (m * m), iy = (sl / m) % m, iz = sl % m;
    const double ox = (ix + 0.5) * sp + wf_uniform_ab(g, -jit, jit);
    const double oy = (iy + 0.5) * sp + wf_uniform_ab(g, -jit, jit);
    const double oz = (iz + 0.5) * sp + wf_uniform_ab(g, -jit, jit);
    const double u1 = wf_uniform(g), u2 = wf_uniform(g), u3 = wf_uniform(g);
    const double tp = 6.283185307179586;
    const double qa = sqrt(1 - u1) * sin(tp * u2), qb = sqrt(1 - u1) * cos(tp * u2),
                 qc = sqrt(u1) * sin(tp * u3), qd = sqrt(u1) * cos(tp * u3);
    const double R[3][3] = {
        {1 - 2 * (qb * qb + qc * qc), 2 * (qa * qb - qc * qd), 2 * (qa * qc + qb * qd)},
        {2 * (qa * qb + qc * qd), 1 - 2 * (qa * qa + qc * qc), 2 * (qb * qc - qa * qd)},
        {2 * (qa * qc - qb * qd), 2 * (qb * qc + qa * qd), 1 - 2 * (qa * qa + qb * qb)}};
    const int64_t o = 3 * w;
    x[o] = wf_wrap(ox, box);
    y[o] = wf_wrap(oy, box);
    z[o] = wf_wrap(oz, box);
    for (int h = 0; h < 2; ++h) {
      double d[3];
      for (int a = 0; a < 3; ++a) d[a] = R[a][0] * hb[h][0] + R[a][1] * hb[h][1] + R[a][2] * hb[h][2];
      x[o + 1 + h] = wf_wrap(ox + d[0], box);
      y[o + 1 + h] = wf_wrap(oy + d[1], box);
      z[o + 1 + h] = wf_wrap(oz + d[2], box);
    }
    for (int k = 0; k < 3; ++k) {
      const int64_t i = o + k;
      const int O = (k == 0);
      if (molecule) molecule[i] = (int32_t)w;
      if (model == 0) {
        charge[i] = O ? -0.834 : 0.417;
        lj_sigma[i] = O ? 3.1507 : 0.0;
        lj_epsilon[i] = O ? 0.1521 : 0.0;
        if (hred_parent) hred_parent[i] = (int32_t)i;
        if (hred_factor) hred_factor[i] = 1.0;
      } else {
        charge[i] = O ? -0.51966 : 0.25983;
        lj_sigma[i] = 0.0;
        lj_epsilon[i] = 0.0;
        if (hred_parent) hred_parent[i] = (int32_t)o;
        if (hred_factor) hred_factor[i] = O ? 1.0 : 0.91;
      }
      hal_r0[i] = O ? 3.405 : 2.655;
      hal_epsilon[i] = O ? 0.110 : 0.0135;
      polarizability[i] = O ? 0.837 : 0.496;
    }
  }
  const int64_t n = 3 * n_mol;
  for (int64_t i = 0; i < n; ++i) { /* multipoles: fixed draw order, drawn for both models */
    const double ct = wf_uniform_ab(g, -1.0, 1.0), ph = 6.283185307179586 * wf_uniform(g);
    const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    const double mag = wf_normal(g, 0.15, 0.03);
    double q[6];
    for (int k = 0; k < 6; ++k) q[k] = wf_normal(g, 0.0, 0.1);
    if (dipole) {
      dipole[3 * i] = model ? mag * st * cos(ph) : 0.0;
      dipole[3 * i + 1] = model ? mag * st * sin(ph) : 0.0;
      dipole[3 * i + 2] = model ? mag * ct : 0.0;
    }
    if (quadrupole) {
      const double tr = (q[0] + q[3] + q[5]) / 3.0;
      double* Q = quadrupole + 6 * i;
      Q[0] = model ? q[0] - tr : 0.0; Q[1] = model ? q[1] : 0.0; Q[2] = model ? q[2] : 0.0;
      Q[3] = model ? q[3] - tr : 0.0; Q[4] = model ? q[4] : 0.0; Q[5] = model ? q[5] - tr : 0.0;
    }
  }
  free(slot);
  free(g);
  return 0;
}

/* proj/src/system.cpp:32-55 */
static void draw_site_params(size_t n, mt64* g, double* charge, double* sig, double* eps,
                             double* r0, double* heps, double* pol) {
  double qsum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double q = mt64_uniform(g, -0.5, 0.5);
    charge[i] = q;
    qsum += q;
    sig[i] = mt64_uniform(g, 0.9, 1.1);
    eps[i] = mt64_uniform(g, 0.5, 1.5);
    r0[i] = mt64_uniform(g, 1.1, 1.3);
    heps[i] = mt64_uniform(g, 0.5, 1.5);
    pol[i] = mt64_uniform(g, 0.5, 1.5);
  }
  if (n > 0) {
    double shift = qsum / (double)n;
    for (size_t i = 0; i < n; ++i) charge[i] -= shift;
  }
}

/* proj/src/system.cpp:65-173 */
int mdo_generate_system(int kind, size_t n, double lx, double ly, double lz, uint64_t seed,
                        double min_sep, double* x, double* y, double* z, double* charge,
                        double* lj_sigma, double* lj_epsilon, double* hal_r0,
                        double* hal_epsilon, double* polarizability) {
  if (!box_ok(lx, ly, lz)) return fail(MDO_CONTRACT, "box edges must be positive and finite");
  if (n < 1) return fail(MDO_CONTRACT, "generate_system: need at least one site");
  mt64 g;
  mt64_seed(&g, seed);
  if (kind == 0) {
    size_t m = 1;
    while (m * m * m < n) ++m;
    const double sx = lx / (double)m, sy = ly / (double)m, sz = lz / (double)m;
    double sp = fmin(sx, fmin(sy, sz));
    const double jitter = 0.05 * sp;
    if (sp - 2.0 * jitter < min_sep)
      return fail(5, "generate_system: lattice too dense for the minimum separation");
    size_t i = 0;
    for (size_t ix = 0; ix < m && i < n; ++ix)
      for (size_t iy = 0; iy < m && i < n; ++iy)
        for (size_t iz = 0; iz < m && i < n; ++iz) {
          { double jx = mt64_uniform(&g, -jitter, jitter); x[i] = wrap_into(((double)ix + 0.5) * sx + jx, lx); }
          { double jy = mt64_uniform(&g, -jitter, jitter); y[i] = wrap_into(((double)iy + 0.5) * sy + jy, ly); }
          { double jz = mt64_uniform(&g, -jitter, jitter); z[i] = wrap_into(((double)iz + 0.5) * sz + jz, lz); }
          ++i;
        }
  } else {
    const double cell = min_sep;
    int gx = (int)(lx / cell), gy = (int)(ly / cell), gz = (int)(lz / cell);
    if (gx < 1) gx = 1;
    if (gy < 1) gy = 1;
    if (gz < 1) gz = 1;
    size_t ncell = (size_t)gx * gy * gz;
    /* bucket lists as linked lists (head per cell, next per site) */
    int32_t* head = (int32_t*)malloc(ncell * sizeof(int32_t));
    int32_t* next = (int32_t*)malloc(n * sizeof(int32_t));
    int32_t* tail = (int32_t*)malloc(ncell * sizeof(int32_t));
    for (size_t c = 0; c < ncell; ++c) head[c] = tail[c] = -1;
    const double sep2 = min_sep * min_sep;
    box_t b = make_box(lx, ly, lz);
    for (size_t i = 0; i < n; ++i) {
      int placed = 0;
      for (int attempt = 0; attempt < 200 && !placed; ++attempt) {
        double px = mt64_uniform(&g, 0.0, lx);
        double py = mt64_uniform(&g, 0.0, ly);
        double pz = mt64_uniform(&g, 0.0, lz);
        px = wrap_into(px, lx);
        py = wrap_into(py, ly);
        pz = wrap_into(pz, lz);
        int clash = 0;
        int cx = (int)(px / lx * gx), cy = (int)(py / ly * gy), cz = (int)(pz / lz * gz);
        if (cx > gx - 1) cx = gx - 1;
        if (cy > gy - 1) cy = gy - 1;
        if (cz > gz - 1) cz = gz - 1;
        for (int ox = -1; ox <= 1 && !clash; ++ox)
          for (int oy = -1; oy <= 1 && !clash; ++oy)
            for (int oz = -1; oz <= 1 && !clash; ++oz) {
              int wx = (cx + ox + gx) % gx, wy = (cy + oy + gy) % gy, wz = (cz + oz + gz) % gz;
              size_t c = ((size_t)wx * gy + wy) * gz + wz;
              for (int32_t j = head[c]; j >= 0; j = next[j]) {
                double dx = mdo_wrap1(px - x[j], b.lx, b.ix, b.hx);
                double dy = mdo_wrap1(py - y[j], b.ly, b.iy, b.hy);
                double dz = mdo_wrap1(pz - z[j], b.lz, b.iz, b.hz);
                if (mdo_dist2(dx, dy, dz) < sep2) {
                  clash = 1;
                  break;
                }
              }
            }
        if (!clash) {
          x[i] = px;
          y[i] = py;
          z[i] = pz;
          size_t c = ((size_t)cx * gy + cy) * gz + cz;
          next[i] = -1;
          if (tail[c] < 0) head[c] = (int32_t)i; else next[tail[c]] = (int32_t)i;
          tail[c] = (int32_t)i;
          placed = 1;
        }
      }
      if (!placed) {
        free(head); free(next); free(tail);
        return fail(5, "generate_system: density too high to respect the minimum separation");
      }
    }
    free(head); free(next); free(tail);
  }
  draw_site_params(n, &g, charge, lj_sigma, lj_epsilon, hal_r0, hal_epsilon, polarizability);
  return MDO_OK;
}

/* proj/src/system.cpp:175-190 */
void mdo_random_dipoles(size_t n, uint64_t seed, double magnitude, double* mx, double* my,
                        double* mz) {
  mt64 g;
  mt64_seed(&g, seed ^ 0x9e3779b97f4a7c15ULL);
  for (size_t i = 0; i < n; ++i) {
    mx[i] = mt64_uniform(&g, -magnitude, magnitude);
    my[i] = mt64_uniform(&g, -magnitude, magnitude);
    mz[i] = mt64_uniform(&g, -magnitude, magnitude);
  }
}

/* ------------------------------------------------------- neighbour table */

static int validate_system(const mdo_system* s) {
  if (!box_ok(s->lx, s->ly, s->lz)) return fail(MDO_CONTRACT, "box edges must be positive and finite");
  /* proj/src/system.cpp:18-27 */
  const double L[3] = {s->lx, s->ly, s->lz};
  const double* p[3] = {s->x, s->y, s->z};
  for (int c = 0; c < 3; ++c)
    for (size_t i = 0; i < s->n; ++i)
      if (!(p[c][i] >= 0.0 && p[c][i] < L[c]))
        return fail(MDO_CONTRACT, "ParticleSystem: position outside the box");
  return MDO_OK;
}

static double min_edge(const mdo_system* s) { return fmin(s->lx, fmin(s->ly, s->lz)); }

static size_t pad_count(size_t n, size_t m) { return (n + m - 1) & ~(m - 1); }

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* proj/src/neighbors_impl.hpp:13-32 */
static int stencil_cells(int ncx, int ncy, int ncz, int32_t cell, int32_t out[27]) {
  const int cz = cell % ncz, cy = (cell / ncz) % ncy, cx = cell / (ncz * ncy);
  int n = 0;
  for (int ox = -1; ox <= 1; ++ox)
    for (int oy = -1; oy <= 1; ++oy)
      for (int oz = -1; oz <= 1; ++oz) {
        int wx = (cx + ox + ncx) % ncx, wy = (cy + oy + ncy) % ncy, wz = (cz + oz + ncz) % ncz;
        out[n++] = (wx * ncy + wy) * ncz + wz;
      }
  qsort(out, (size_t)n, sizeof(int32_t), cmp_i32);
  int u = 0;
  for (int k = 0; k < n; ++k)
    if (u == 0 || out[k] != out[u - 1]) out[u++] = out[k];
  return u;
}

/* proj/src/neighbors.cpp:10-36 (grid) + neighbors_vec.cpp:8-94 (table) +
 * neighbors.cpp:90-113 (finalize). Pair order within a segment is the
 * reference's: stencil cells ascending, bucket (index) order inside a cell. */
int mdo_table_build(const mdo_system* s, double list_cutoff, size_t extra_pad, mdo_table* out) {
  memset(out, 0, sizeof *out);
  int rc = validate_system(s);
  if (rc) return rc;
  if (!(list_cutoff > 0) || !isfinite(list_cutoff))
    return fail(MDO_CONTRACT, "build_cell_grid: cutoff must be positive");
  if (list_cutoff > 0.5 * min_edge(s))
    return fail(MDO_CONTRACT, "build_cell_grid: cutoff exceeds half the smallest box edge");
  if (extra_pad % 16 != 0)
    return fail(MDO_CONTRACT, "build_neighbor_table: extra padding must be a multiple of 16");
  const size_t n = s->n;
  int ncx = (int)(s->lx / list_cutoff), ncy = (int)(s->ly / list_cutoff),
      ncz = (int)(s->lz / list_cutoff);
  if (ncx < 1) ncx = 1;
  if (ncy < 1) ncy = 1;
  if (ncz < 1) ncz = 1;
  const double ex = s->lx / ncx, ey = s->ly / ncy, ez = s->lz / ncz;
  const size_t ncell = (size_t)ncx * ncy * ncz;
  int32_t* cell_of = (int32_t*)malloc(n * sizeof(int32_t));
  size_t* cstart = (size_t*)calloc(ncell + 1, sizeof(size_t));
  int32_t* bucket = (int32_t*)malloc(n * sizeof(int32_t));
  for (size_t i = 0; i < n; ++i) {
    int cx = (int)(s->x[i] / ex), cy = (int)(s->y[i] / ey), cz = (int)(s->z[i] / ez);
    if (cx > ncx - 1) cx = ncx - 1;
    if (cy > ncy - 1) cy = ncy - 1;
    if (cz > ncz - 1) cz = ncz - 1;
    cell_of[i] = (cx * ncy + cy) * ncz + cz;
    cstart[cell_of[i] + 1]++;
  }
  for (size_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
  {
    size_t* fillp = (size_t*)malloc(ncell * sizeof(size_t));
    memcpy(fillp, cstart, ncell * sizeof(size_t));
    for (size_t i = 0; i < n; ++i) bucket[fillp[cell_of[i]]++] = (int32_t)i;
    free(fillp);
  }
  /* neighbors.cpp:83-87 */
  if (list_cutoff > fmin(ex, fmin(ey, ez)) + 1e-12) {
    free(cell_of); free(cstart); free(bucket);
    return fail(MDO_CONTRACT, "neighbor table: cell edge smaller than the list cutoff");
  }
  const double c2 = list_cutoff * list_cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  out->n_sites = n;
  out->cutoff = list_cutoff;
  out->nnvlst = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  out->nvloop8 = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  out->nvloop16 = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  out->offset = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  size_t cap = 1024, total = 0;
  int32_t* packed = (int32_t*)malloc(cap * sizeof(int32_t));
  int32_t* found = (int32_t*)malloc((n ? n : 1) * sizeof(int32_t));
  int32_t cells[27];
  for (size_t i = 0; i < n; ++i) {
    size_t kept = 0;
    int nc = stencil_cells(ncx, ncy, ncz, cell_of[i], cells);
    for (int c = 0; c < nc; ++c)
      for (size_t q = cstart[cells[c]]; q < cstart[cells[c] + 1]; ++q) {
        int32_t j = bucket[q];
        if (j <= (int32_t)i) continue;
        double dx, dy, dz;
        if (pair_d(s, &b, i, (size_t)j, &dx, &dy, &dz) <= c2) found[kept++] = j;
      }
    if (kept > MDO_MAX_NEIGHBORS) {
      char msg[160];
      snprintf(msg, sizeof msg,
               "neighbor table: site %zu exceeds the per-site neighbor capacity", i);
      free(cell_of); free(cstart); free(bucket); free(packed); free(found);
      mdo_table_free(out);
      return fail(MDO_CAPACITY, msg);
    }
    size_t nv16 = pad_count(kept, 16) + extra_pad;
    out->nnvlst[i] = (uint32_t)kept;
    out->nvloop8[i] = (uint32_t)(pad_count(kept, 8) + extra_pad);
    out->nvloop16[i] = (uint32_t)nv16;
    out->offset[i] = total;
    while (total + nv16 > cap) {
      cap *= 2;
      packed = (int32_t*)realloc(packed, cap * sizeof(int32_t));
    }
    int32_t sentinel = kept > 0 ? found[kept - 1] : 0;
    for (size_t k = 0; k < nv16; ++k) packed[total + k] = k < kept ? found[k] : sentinel;
    total += nv16;
  }
  out->indices = packed;
  out->total = total;
  out->scale = (double*)malloc((total ? total : 1) * sizeof(double));
  for (size_t i = 0; i < n; ++i)
    for (uint32_t k = 0; k < out->nvloop16[i]; ++k)
      out->scale[out->offset[i] + k] = k < out->nnvlst[i] ? 1.0 : 0.0;
  free(cell_of); free(cstart); free(bucket); free(found);
  return MDO_OK;
}

void mdo_table_free(mdo_table* t) {
  free(t->nnvlst); free(t->nvloop8); free(t->nvloop16); free(t->offset);
  free(t->indices); free(t->scale);
  memset(t, 0, sizeof *t);
}

/* proj/src/neighbors.cpp:38-57 */
int mdo_brute_force_pairs(const mdo_system* s, double cutoff, int32_t* out, size_t cap,
                          size_t* npairs) {
  int rc = validate_system(s);
  if (rc) return rc;
  if (!(cutoff > 0) || cutoff > 0.5 * min_edge(s))
    return fail(MDO_CONTRACT, "brute_force_pairs: invalid cutoff");
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  size_t np = 0;
  for (size_t i = 0; i < s->n; ++i)
    for (size_t j = i + 1; j < s->n; ++j) {
      double dx, dy, dz;
      if (pair_d(s, &b, i, j, &dx, &dy, &dz) <= c2) {
        if (np < cap) {
          out[2 * np] = (int32_t)i;
          out[2 * np + 1] = (int32_t)j;
        }
        ++np;
      }
    }
  *npairs = np;
  return np > cap ? fail(MDO_CAPACITY, "brute_force_pairs: output capacity") : MDO_OK;
}

static int cmp_pair(const void* a, const void* b) {
  const int32_t* p = (const int32_t*)a;
  const int32_t* q = (const int32_t*)b;
  if (p[0] != q[0]) return (p[0] > q[0]) - (p[0] < q[0]);
  return (p[1] > q[1]) - (p[1] < q[1]);
}

/* proj/src/neighbors.cpp:59-72 */
int mdo_table_pairs(const mdo_table* t, int32_t* out, size_t cap, size_t* npairs) {
  size_t np = 0;
  for (size_t i = 0; i < t->n_sites; ++i) np += t->nnvlst[i];
  *npairs = np;
  if (np > cap) return fail(MDO_CAPACITY, "table_pairs: output capacity");
  size_t k = 0;
  for (size_t i = 0; i < t->n_sites; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    for (uint32_t q = 0; q < t->nnvlst[i]; ++q) {
      int32_t a = (int32_t)i, bb = idx[q];
      out[2 * k] = a < bb ? a : bb;
      out[2 * k + 1] = a < bb ? bb : a;
      ++k;
    }
  }
  qsort(out, np, 2 * sizeof(int32_t), cmp_pair);
  return MDO_OK;
}

/* ------------------------------------------------------- pair kernels */

/* proj/src/kernels_impl.hpp:8-20 */
static int validate_kernel(const mdo_system* s, const mdo_table* t, double cutoff) {
  if (t->n_sites != s->n) return fail(MDO_CONTRACT, "kernel: table does not match the system");
  if (!(cutoff > 0) || cutoff > t->cutoff)
    return fail(MDO_CONTRACT, "kernel: cutoff must be positive and within the list cutoff");
  return MDO_OK;
}

static inline int excluded(const mdo_system* s, int exclude, size_t i, size_t j) {
  return exclude && s->molecule && s->molecule[i] == s->molecule[j];
}

static void zero3(size_t n, double* a, double* b, double* c) {
  memset(a, 0, n * sizeof(double));
  memset(b, 0, n * sizeof(double));
  memset(c, 0, n * sizeof(double));
}

static inline void add_virial(double* w, double dx, double dy, double dz, double fx,
                              double fy, double fz) {
  w[0] += dx * fx; w[1] += dx * fy; w[2] += dx * fz;
  w[3] += dy * fx; w[4] += dy * fy; w[5] += dy * fz;
  w[6] += dz * fx; w[7] += dz * fy; w[8] += dz * fz;
}

/* proj/include/mdvec/kernels.hpp:42-48 */
static void lj_core(double r2, double sij, double eij, double* u, double* fs) {
  const double inv_r2 = 1.0 / r2;
  const double s2 = sij * sij * inv_r2;
  const double s6 = s2 * s2 * s2;
  const double s12 = s6 * s6;
  *u = 4.0 * eij * (s12 - s6);
  *fs = 24.0 * eij * (2.0 * s12 - s6) * inv_r2;
}

/* proj/src/kernels_scalar.cpp:10-51 */
int mdo_lj(const mdo_system* s, const mdo_table* t, double cutoff, int shift, int exclude,
           double* fx, double* fy, double* fz, double* energy, double* virial) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  zero3(s->n, fx, fy, fz);
  double w[9] = {0};
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  double e = 0.0;
  for (size_t i = 0; i < s->n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    double fxi = 0, fyi = 0, fzi = 0;
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double dx, dy, dz;
      const double r2 = pair_d(s, &b, i, j, &dx, &dy, &dz);
      if (r2 <= c2 && !excluded(s, exclude, i, j)) {
        if (!(r2 > 0)) return fail(MDO_SINGULARITY, "lj_pair: zero separation");
        const double sij = 0.5 * (s->lj_sigma[i] + s->lj_sigma[j]);
        const double eij = sqrt(s->lj_epsilon[i] * s->lj_epsilon[j]);
        double u, fs, uc, fc;
        lj_core(r2, sij, eij, &u, &fs);
        if (shift) {
          lj_core(c2, sij, eij, &uc, &fc);
          u -= uc;
        }
        e += u;
        const double px = fs * dx, py = fs * dy, pz = fs * dz;
        fxi += px; fyi += py; fzi += pz;
        fx[j] -= px; fy[j] -= py; fz[j] -= pz;
        add_virial(w, dx, dy, dz, px, py, pz);
      }
    }
    fx[i] += fxi; fy[i] += fyi; fz[i] += fzi;
  }
  *energy = e;
  if (virial) memcpy(virial, w, sizeof w);
  return MDO_OK;
}

/* proj/src/kernels_scalar.cpp:53-94, pair core kernels.hpp:57-64 */
int mdo_ewald_real(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                   double electric, int exclude, double* fx, double* fy, double* fz,
                   double* energy, double* virial) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  if (alpha < 0) return fail(MDO_CONTRACT, "ewald: alpha must be nonnegative");
  zero3(s->n, fx, fy, fz);
  double w[9] = {0};
  const double c2 = cutoff * cutoff;
  const double two_over_sqrt_pi = 1.1283791670955126;
  box_t b = make_box(s->lx, s->ly, s->lz);
  double e = 0.0;
  for (size_t i = 0; i < s->n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    double fxi = 0, fyi = 0, fzi = 0;
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double dx, dy, dz;
      const double r2 = pair_d(s, &b, i, j, &dx, &dy, &dz);
      if (r2 <= c2 && !excluded(s, exclude, i, j)) {
        const double r = sqrt(r2);
        if (!(r > 0)) return fail(MDO_SINGULARITY, "ewald_real_pair: zero separation");
        const double qq = electric * s->charge[i] * s->charge[j];
        const double inv_r = 1.0 / r;
        const double ee = erfc(alpha * r) * inv_r;
        const double g = alpha * two_over_sqrt_pi * exp(-alpha * alpha * r * r);
        const double u = qq * ee;
        const double fs = qq * (ee + g) * inv_r * inv_r;
        e += u;
        const double px = fs * dx, py = fs * dy, pz = fs * dz;
        fxi += px; fyi += py; fzi += pz;
        fx[j] -= px; fy[j] -= py; fz[j] -= pz;
        add_virial(w, dx, dy, dz, px, py, pz);
      }
    }
    fx[i] += fxi; fy[i] += fyi; fz[i] += fzi;
  }
  *energy = e;
  if (virial) memcpy(virial, w, sizeof w);
  return MDO_OK;
}

/* proj/include/mdvec/polar.hpp:26-41 */
static void halgren_core(double rho, double eij, double delta, double gamma, double* u,
                         double* dudrho) {
  const double t1 = (1.0 + delta) / (rho + delta);
  const double t2 = t1 * t1;
  const double t4 = t2 * t2;
  const double t7 = t4 * t2 * t1;
  const double rho2 = rho * rho;
  const double rho3 = rho2 * rho;
  const double rho6 = rho3 * rho3;
  const double rho7 = rho6 * rho;
  const double g1 = (1.0 + gamma) / (rho7 + gamma);
  const double bb = g1 - 2.0;
  *u = eij * t7 * bb;
  *dudrho = -7.0 * eij * t7 * (bb / (rho + delta) + rho6 * g1 / (rho7 + gamma));
}

/* proj/src/polar_scalar.cpp:26-67 */
int mdo_halgren(const mdo_system* s, const mdo_table* t, double cutoff, double delta,
                double gamma, int exclude, double* fx, double* fy, double* fz,
                double* energy, double* virial) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  zero3(s->n, fx, fy, fz);
  double w[9] = {0};
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  double e = 0.0;
  for (size_t i = 0; i < s->n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    double fxi = 0, fyi = 0, fzi = 0;
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double dx, dy, dz;
      const double r2 = pair_d(s, &b, i, j, &dx, &dy, &dz);
      if (r2 <= c2 && !excluded(s, exclude, i, j)) {
        const double r = sqrt(r2);
        const double r0 = 0.5 * (s->hal_r0[i] + s->hal_r0[j]);
        const double eij = sqrt(s->hal_epsilon[i] * s->hal_epsilon[j]);
        const double rho = r / r0;
        if (!(rho > 0)) return fail(MDO_SINGULARITY, "halgren_pair: zero separation");
        double u, dudrho;
        halgren_core(rho, eij, delta, gamma, &u, &dudrho);
        e += u;
        const double fs = -dudrho / (r0 * r);
        const double px = fs * dx, py = fs * dy, pz = fs * dz;
        fxi += px; fyi += py; fzi += pz;
        fx[j] -= px; fy[j] -= py; fz[j] -= pz;
        add_virial(w, dx, dy, dz, px, py, pz);
      }
    }
    fx[i] += fxi; fy[i] += fyi; fz[i] += fzi;
  }
  *energy = e;
  if (virial) memcpy(virial, w, sizeof w);
  return MDO_OK;
}

/* proj/include/mdvec/polar.hpp:55-62 */
static void thole_core(double r, double ai, double aj, double a, double* l3, double* l5,
                       double* l7) {
  const double u = r / cbrt(sqrt(ai * aj));
  const double au3 = a * u * u * u;
  const double ex = exp(-au3);
  *l3 = 1.0 - ex;
  *l5 = 1.0 - (1.0 + au3) * ex;
  if (l7) *l7 = 1.0 - (1.0 + au3 + 0.6 * au3 * au3) * ex; /* EXTENSION (Thole lambda7) */
}

/* proj/src/polar_scalar.cpp:69-118 */
int mdo_tmatvec_thole(const mdo_system* s, const mdo_table* t, double cutoff, double thole_a,
                      const double* mx, const double* my, const double* mz, double* ex,
                      double* ey, double* ez) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  zero3(s->n, ex, ey, ez);
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  for (size_t i = 0; i < s->n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    const double ai = s->polarizability[i];
    double exi = 0, eyi = 0, ezi = 0;
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double dx, dy, dz;
      const double r2 = pair_d(s, &b, i, j, &dx, &dy, &dz);
      if (r2 <= c2) {
        if (!(r2 > 0)) return fail(MDO_SINGULARITY, "dipole_field_matvec: coincident sites");
        const double r = sqrt(r2);
        double l3, l5;
        thole_core(r, ai, s->polarizability[j], thole_a, &l3, &l5, NULL);
        const double r3 = r2 * r, r5 = r3 * r2;
        const double rr3 = l3 / r3, rr5 = 3.0 * l5 / r5;
        const double dotj = mx[j] * dx + my[j] * dy + mz[j] * dz;
        exi += rr5 * dotj * dx - rr3 * mx[j];
        eyi += rr5 * dotj * dy - rr3 * my[j];
        ezi += rr5 * dotj * dz - rr3 * mz[j];
        const double doti = mx[i] * dx + my[i] * dy + mz[i] * dz;
        ex[j] += rr5 * doti * dx - rr3 * mx[i];
        ey[j] += rr5 * doti * dy - rr3 * my[i];
        ez[j] += rr5 * doti * dz - rr3 * mz[i];
      }
    }
    ex[i] += exi; ey[i] += eyi; ez[i] += ezi;
  }
  return MDO_OK;
}

/* proj/src/polar_scalar.cpp:120-159 */
int mdo_perm_field_thole(const mdo_system* s, const mdo_table* t, double cutoff,
                         double thole_a, double* ex, double* ey, double* ez) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  zero3(s->n, ex, ey, ez);
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  for (size_t i = 0; i < s->n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    const double ai = s->polarizability[i], qi = s->charge[i];
    double exi = 0, eyi = 0, ezi = 0;
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double dx, dy, dz;
      const double r2 = pair_d(s, &b, i, j, &dx, &dy, &dz);
      if (r2 <= c2) {
        if (!(r2 > 0)) return fail(MDO_SINGULARITY, "permanent_field: coincident sites");
        const double r = sqrt(r2);
        double l3, l5;
        thole_core(r, ai, s->polarizability[j], thole_a, &l3, &l5, NULL);
        const double c = l3 / (r2 * r);
        const double qj = s->charge[j];
        exi += c * qj * dx; eyi += c * qj * dy; ezi += c * qj * dz;
        ex[j] -= c * qi * dx; ey[j] -= c * qi * dy; ez[j] -= c * qi * dz;
      }
    }
    ex[i] += exi; ey[i] += eyi; ez[i] += ezi;
  }
  return MDO_OK;
}

/* proj/src/polar_scalar.cpp:161-198 */
int mdo_jacobi(const mdo_system* s, const mdo_table* t, double cutoff, double thole_a,
               double tol, size_t max_iter, double* mx, double* my, double* mz,
               double* last_residual, size_t* iters) {
  if (!(tol > 0)) return fail(MDO_CONTRACT, "jacobi_polarization_solve: tol must be positive");
  if (max_iter < 1) return fail(MDO_CONTRACT, "jacobi_polarization_solve: max_iter must be >= 1");
  const size_t n = s->n;
  double* ep = (double*)malloc(3 * n * sizeof(double) + 1);
  double* tm = (double*)malloc(3 * n * sizeof(double) + 1);
  int rc = mdo_perm_field_thole(s, t, cutoff, thole_a, ep, ep + n, ep + 2 * n);
  if (rc) { free(ep); free(tm); return rc; }
  memset(mx, 0, n * sizeof(double));
  memset(my, 0, n * sizeof(double));
  memset(mz, 0, n * sizeof(double));
  double resid = 0.0;
  for (size_t it = 0; it < max_iter; ++it) {
    rc = mdo_tmatvec_thole(s, t, cutoff, thole_a, mx, my, mz, tm, tm + n, tm + 2 * n);
    if (rc) { free(ep); free(tm); return rc; }
    resid = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double ai = s->polarizability[i];
      const double nx = ai * (ep[i] + tm[i]);
      const double ny = ai * (ep[n + i] + tm[n + i]);
      const double nz = ai * (ep[2 * n + i] + tm[2 * n + i]);
      resid = fmax(resid, fabs(nx - mx[i]));
      resid = fmax(resid, fabs(ny - my[i]));
      resid = fmax(resid, fabs(nz - mz[i]));
      mx[i] = nx; my[i] = ny; mz[i] = nz;
    }
    *iters = it + 1;
    *last_residual = resid;
    if (resid <= tol) { free(ep); free(tm); return MDO_OK; }
  }
  free(ep); free(tm);
  return fail(MDO_CONVERGENCE, "jacobi_polarization_solve: no convergence after max_iter");
}

/* ============================================================ EXTENSIONS */

/* wrap_into without contraction: p - L*floor(p/L), then [0, L) clamp.
 * Device twin: csrc reduce-sites kernel (same separately rounded ops). */
static double wrap_into_exact(double p, double L) {
  double k = floor(p / L);
  double m = L * k;
  p = p - m;
  if (p >= L) p = 0.0;
  if (p < 0.0) p = 0.0;
  return p;
}

void mdo_reduce_sites(size_t n, const double* x, const double* y, const double* z,
                      const int32_t* parent, const double* factor, double lx, double ly,
                      double lz, double* xr, double* yr, double* zr) {
  box_t b = make_box(lx, ly, lz);
  for (size_t i = 0; i < n; ++i) {
    const size_t p = (size_t)parent[i];
    if (p == i) { xr[i] = x[i]; yr[i] = y[i]; zr[i] = z[i]; continue; }
    const double f = factor[i];
    const double dx = mdo_wrap1(x[i] - x[p], b.lx, b.ix, b.hx);
    const double dy = mdo_wrap1(y[i] - y[p], b.ly, b.iy, b.hy);
    const double dz = mdo_wrap1(z[i] - z[p], b.lz, b.iz, b.hz);
    const double sx = f * dx, sy = f * dy, sz = f * dz;
    xr[i] = wrap_into_exact(x[p] + sx, lx);
    yr[i] = wrap_into_exact(y[p] + sy, ly);
    zr[i] = wrap_into_exact(z[p] + sz, lz);
  }
}

void mdo_reduce_forces(size_t n, const int32_t* parent, const double* factor,
                       const double* frx, const double* fry, const double* frz, double* fx,
                       double* fy, double* fz) {
  zero3(n, fx, fy, fz);
  for (size_t i = 0; i < n; ++i) {
    const size_t p = (size_t)parent[i];
    if (p == i) { fx[i] += frx[i]; fy[i] += fry[i]; fz[i] += frz[i]; continue; }
    const double f = factor[i], g = 1.0 - factor[i];
    fx[i] += f * frx[i]; fy[i] += f * fry[i]; fz[i] += f * frz[i];
    fx[p] += g * frx[i]; fy[p] += g * fry[i]; fz[p] += g * frz[i];
  }
}

/* Tinker bn recursion: B0 = erfc(a r)/r,
 * Bn = ((2n-1) B(n-1) + (2a^2)^n/(a sqrt(pi)) exp(-a^2 r^2)) / r^2.
 * At alpha = 0, Bn = (2n-1)!!/r^(2n+1). */
void mdo_ewald_bn(double r, double alpha, int nmax, double* bn) {
  const double sqrtpi = 1.7724538509055160273;
  const double r2 = r * r;
  bn[0] = erfc(alpha * r) / r;
  const double alsq2 = 2.0 * alpha * alpha;
  double alsq2n = alpha > 0 ? 1.0 / (sqrtpi * alpha) : 0.0;
  const double exp2a = exp(-alpha * alpha * r2);
  for (int k = 1; k <= nmax; ++k) {
    alsq2n *= alsq2;
    bn[k] = ((double)(2 * k - 1) * bn[k - 1] + alsq2n * exp2a) / r2;
  }
}

static void bare_bn(double r, int nmax, double* g) {
  const double r2 = r * r;
  g[0] = 1.0 / r;
  for (int k = 1; k <= nmax; ++k) g[k] = (double)(2 * k - 1) * g[k - 1] / r2;
}

int mdo_tmatvec_ewald(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                      double thole_a, const double* mu, double* e) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  const size_t n = s->n;
  memset(e, 0, 3 * n * sizeof(double));
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double d[3];
      const double r2 = pair_d(s, &b, i, j, &d[0], &d[1], &d[2]);
      if (!(r2 <= c2)) continue;
      if (!(r2 > 0)) return fail(MDO_SINGULARITY, "tmatvec: coincident sites");
      const double r = sqrt(r2);
      double bn[3], g[3], l3, l5;
      mdo_ewald_bn(r, alpha, 2, bn);
      bare_bn(r, 2, g);
      thole_core(r, s->polarizability[i], s->polarizability[j], thole_a, &l3, &l5, NULL);
      const double rr3 = bn[1] - (1.0 - l3) * g[1];
      const double rr5 = bn[2] - (1.0 - l5) * g[2];
      const double* mj = mu + 3 * j;
      const double* mi = mu + 3 * i;
      const double dotj = mj[0] * d[0] + mj[1] * d[1] + mj[2] * d[2];
      const double doti = mi[0] * d[0] + mi[1] * d[1] + mi[2] * d[2];
      for (int a = 0; a < 3; ++a) {
        e[3 * i + a] += rr5 * dotj * d[a] - rr3 * mj[a];
        e[3 * j + a] += rr5 * doti * d[a] - rr3 * mi[a];
      }
    }
  }
  return MDO_OK;
}

/* unpack the 6-component traceless quadrupole into a symmetric 3x3 */
static void quad3(const double* q6, double Q[3][3]) {
  Q[0][0] = q6[0]; Q[0][1] = Q[1][0] = q6[1]; Q[0][2] = Q[2][0] = q6[2];
  Q[1][1] = q6[3]; Q[1][2] = Q[2][1] = q6[4]; Q[2][2] = q6[5];
}

/* field at site `at` from the multipole of site `src`, R = r_at - r_src:
 * E = R (rr3 q + rr5 mu.R + rr7 R.Q.R) - rr3 mu - 2 rr5 Q R */
static void mpole_field_at(double q, const double* mu, double Q[3][3], const double R[3],
                           double rr3, double rr5, double rr7, double* E) {
  double QR[3];
  for (int a = 0; a < 3; ++a) QR[a] = Q[a][0] * R[0] + Q[a][1] * R[1] + Q[a][2] * R[2];
  const double mr = mu[0] * R[0] + mu[1] * R[1] + mu[2] * R[2];
  const double rqr = R[0] * QR[0] + R[1] * QR[1] + R[2] * QR[2];
  const double c = rr3 * q + rr5 * mr + rr7 * rqr;
  for (int a = 0; a < 3; ++a) E[a] += c * R[a] - rr3 * mu[a] - 2.0 * rr5 * QR[a];
}

static const double zero6[6] = {0, 0, 0, 0, 0, 0};
static const double zero3v[3] = {0, 0, 0};

int mdo_perm_field_ewald(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                         double thole_a, int exclude, double* e) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  const size_t n = s->n;
  memset(e, 0, 3 * n * sizeof(double));
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double d[3];
      const double r2 = pair_d(s, &b, i, j, &d[0], &d[1], &d[2]);
      if (!(r2 <= c2) || excluded(s, exclude, i, j)) continue;
      if (!(r2 > 0)) return fail(MDO_SINGULARITY, "perm_field: coincident sites");
      const double r = sqrt(r2);
      double bn[4], g[4], l3, l5, l7;
      mdo_ewald_bn(r, alpha, 3, bn);
      bare_bn(r, 3, g);
      thole_core(r, s->polarizability[i], s->polarizability[j], thole_a, &l3, &l5, &l7);
      const double rr3 = bn[1] - (1.0 - l3) * g[1];
      const double rr5 = bn[2] - (1.0 - l5) * g[2];
      const double rr7 = bn[3] - (1.0 - l7) * g[3];
      double Qi[3][3], Qj[3][3];
      quad3(s->quadrupole ? s->quadrupole + 6 * i : zero6, Qi);
      quad3(s->quadrupole ? s->quadrupole + 6 * j : zero6, Qj);
      const double* mi = s->dipole ? s->dipole + 3 * i : zero3v;
      const double* mj = s->dipole ? s->dipole + 3 * j : zero3v;
      double Rj[3] = {-d[0], -d[1], -d[2]};
      mpole_field_at(s->charge[j], mj, Qj, d, rr3, rr5, rr7, e + 3 * i);
      mpole_field_at(s->charge[i], mi, Qi, Rj, rr3, rr5, rr7, e + 3 * j);
    }
  }
  return MDO_OK;
}

/* ---- generic Cartesian interaction tensors --------------------------------
 * T^(k)_{a1..ak}(r) = d^k G0 / dr_a1..dr_ak with dG_n/dr_a = -r_a G_{n+1}:
 * T^(k) = sum_p (-1)^(k-p) G_{k-p} sum_{p disjoint index pairs} prod delta prod r. */
static double tens_rec(const int* idx, int k, const double* r, int used_mask, int npairs,
                       const double* G) {
  /* find first unused index */
  int first = -1;
  for (int a = 0; a < k; ++a)
    if (!(used_mask & (1 << a))) { first = a; break; }
  if (first < 0) {
    /* all indices consumed by pairs */
    const int m = k - npairs; /* G index: k - p */
    const double sign = ((k - npairs) % 2) ? -1.0 : 1.0;
    return sign * G[m];
  }
  double total = 0.0;
  /* option 1: index `first` is a free r factor */
  {
    /* it stays unpaired: multiply r and continue with remaining */
    double sub = tens_rec(idx, k, r, used_mask | (1 << first), npairs, G);
    total += r[idx[first]] * sub;
  }
  /* option 2: pair `first` with a later unused index b */
  for (int b2 = first + 1; b2 < k; ++b2) {
    if (used_mask & (1 << b2)) continue;
    if (idx[first] != idx[b2]) continue;
    total += tens_rec(idx, k, r, used_mask | (1 << first) | (1 << b2), npairs + 1, G);
  }
  return total;
}

static double tensor_elem(int k, const int* idx, const double* r, const double* G) {
  return tens_rec(idx, k, r, 0, 0, G);
}

/* all tensors rank 0..5 */
typedef struct {
  double t0, t1[3], t2[9], t3[27], t4[81], t5[243];
} tens_t;

static void build_tensors(const double* r, const double* G, tens_t* T) {
  int idx[5];
  T->t0 = G[0];
  for (int a = 0; a < 3; ++a) { idx[0] = a; T->t1[a] = tensor_elem(1, idx, r, G); }
  for (int e = 0; e < 9; ++e) {
    idx[0] = e / 3; idx[1] = e % 3;
    T->t2[e] = tensor_elem(2, idx, r, G);
  }
  for (int e = 0; e < 27; ++e) {
    idx[0] = e / 9; idx[1] = (e / 3) % 3; idx[2] = e % 3;
    T->t3[e] = tensor_elem(3, idx, r, G);
  }
  for (int e = 0; e < 81; ++e) {
    idx[0] = e / 27; idx[1] = (e / 9) % 3; idx[2] = (e / 3) % 3; idx[3] = e % 3;
    T->t4[e] = tensor_elem(4, idx, r, G);
  }
  for (int e = 0; e < 243; ++e) {
    idx[0] = e / 81; idx[1] = (e / 27) % 3; idx[2] = (e / 9) % 3; idx[3] = (e / 3) % 3;
    idx[4] = e % 3;
    T->t5[e] = tensor_elem(5, idx, r, G);
  }
}

/* U = (q_i + mu_i.d + Q_i:dd)(q_j - mu_j.d + Q_j:dd) G0(r), r = r_i - r_j.
 * `off` selects the derivative tensors: off=0 energy (ranks 0..4),
 * off=1 gradient component e (ranks 1..5, extra trailing index e). */
static double pair_energy_tensor(double qi, const double* mi, double Qi[3][3], double qj,
                                 const double* mj, double Qj[3][3], const tens_t* T, int off,
                                 int e) {
  /* accessor for T^(k+off) with trailing index e when off=1 */
#define TK0() (off ? T->t1[e] : T->t0)
#define TK1(a) (off ? T->t2[(a) * 3 + e] : T->t1[a])
#define TK2(a, b) (off ? T->t3[((a) * 3 + (b)) * 3 + e] : T->t2[(a) * 3 + (b)])
#define TK3(a, b, c) (off ? T->t4[(((a) * 3 + (b)) * 3 + (c)) * 3 + e] : T->t3[((a) * 3 + (b)) * 3 + (c)])
#define TK4(a, b, c, d) (off ? T->t5[((((a) * 3 + (b)) * 3 + (c)) * 3 + (d)) * 3 + e] : T->t4[(((a) * 3 + (b)) * 3 + (c)) * 3 + (d)])
  double u = qi * qj * TK0();
  for (int c = 0; c < 3; ++c) u += -qi * mj[c] * TK1(c) + mi[c] * qj * TK1(c);
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      u += qi * Qj[a][c] * TK2(a, c) + Qi[a][c] * qj * TK2(a, c);
      u += -mi[a] * mj[c] * TK2(a, c);
    }
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) {
        u += mi[a] * Qj[c][d] * TK3(a, c, d);
        u += -Qi[a][c] * mj[d] * TK3(a, c, d);
      }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) u += Qi[a][b] * Qj[c][d] * TK4(a, b, c, d);
  return u;
#undef TK0
#undef TK1
#undef TK2
#undef TK3
#undef TK4
}

/* dU/dmu_i (vector) and dU/dQ_i (matrix, as U is written with Q_i[a][b]) */
static void pair_grad_i(double qj, const double* mj, double Qj[3][3], const tens_t* T,
                        double gmu[3], double gQ[3][3]) {
  for (int a = 0; a < 3; ++a) {
    double v = qj * T->t1[a];
    for (int c = 0; c < 3; ++c) v += -mj[c] * T->t2[a * 3 + c];
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) v += Qj[c][d] * T->t3[(a * 3 + c) * 3 + d];
    gmu[a] = v;
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double v = qj * T->t2[a * 3 + b];
      for (int c = 0; c < 3; ++c) v += -mj[c] * T->t3[(a * 3 + b) * 3 + c];
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) v += Qj[c][d] * T->t4[((a * 3 + b) * 3 + c) * 3 + d];
      gQ[a][b] = v;
    }
}

/* torque = -dU/dtheta for an infinitesimal rotation of site i's multipoles:
 * d mu = dtheta x mu, dQ = W Q - Q W with (W^a)_bc = eps_bac. */
static void torque_from_grads(const double* mu, double Q[3][3], const double gmu[3],
                              double gQ[3][3], double tau[3]) {
  static const int eps[3][3][3] = {
      {{0, 0, 0}, {0, 0, 1}, {0, -1, 0}},
      {{0, 0, -1}, {0, 0, 0}, {1, 0, 0}},
      {{0, 1, 0}, {-1, 0, 0}, {0, 0, 0}}};
  for (int a = 0; a < 3; ++a) {
    /* dipole: dU = gmu . (e_a x mu) */
    double cross[3];
    for (int b = 0; b < 3; ++b) {
      double v = 0;
      for (int c = 0; c < 3; ++c) v += eps[b][a][c] * mu[c];
      cross[b] = v;
    }
    double du = gmu[0] * cross[0] + gmu[1] * cross[1] + gmu[2] * cross[2];
    /* quadrupole */
    double W[3][3];
    for (int b = 0; b < 3; ++b)
      for (int c = 0; c < 3; ++c) W[b][c] = eps[b][a][c];
    for (int b = 0; b < 3; ++b)
      for (int c = 0; c < 3; ++c) {
        double dq = 0;
        for (int m = 0; m < 3; ++m) dq += W[b][m] * Q[m][c] - Q[b][m] * W[m][c];
        du += gQ[b][c] * dq;
      }
    tau[a] = -du;
  }
}

int mdo_mpole(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
              double electric, int exclude, double* f, double* torque, double* energy,
              double* virial) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  if (alpha < 0) return fail(MDO_CONTRACT, "mpole: alpha must be nonnegative");
  const size_t n = s->n;
  memset(f, 0, 3 * n * sizeof(double));
  memset(torque, 0, 3 * n * sizeof(double));
  double w[9] = {0};
  double etot = 0.0;
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  tens_t T;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double d[3];
      const double r2 = pair_d(s, &b, i, j, &d[0], &d[1], &d[2]);
      if (!(r2 <= c2) || excluded(s, exclude, i, j)) continue;
      if (!(r2 > 0)) return fail(MDO_SINGULARITY, "mpole: coincident sites");
      const double r = sqrt(r2);
      double G[6];
      mdo_ewald_bn(r, alpha, 5, G);
      build_tensors(d, G, &T);
      double Qi[3][3], Qj[3][3];
      quad3(s->quadrupole ? s->quadrupole + 6 * i : zero6, Qi);
      quad3(s->quadrupole ? s->quadrupole + 6 * j : zero6, Qj);
      const double* mi = s->dipole ? s->dipole + 3 * i : zero3v;
      const double* mj = s->dipole ? s->dipole + 3 * j : zero3v;
      const double qi = s->charge[i], qj = s->charge[j];
      etot += electric * pair_energy_tensor(qi, mi, Qi, qj, mj, Qj, &T, 0, 0);
      double fi[3];
      for (int e = 0; e < 3; ++e) {
        fi[e] = -electric * pair_energy_tensor(qi, mi, Qi, qj, mj, Qj, &T, 1, e);
        f[3 * i + e] += fi[e];
        f[3 * j + e] -= fi[e];
      }
      add_virial(w, d[0], d[1], d[2], fi[0], fi[1], fi[2]);
      /* torques: site i directly; site j via the swapped pair at -r */
      double gmu[3], gQ[3][3], tau[3];
      pair_grad_i(qj, mj, Qj, &T, gmu, gQ);
      torque_from_grads(mi, Qi, gmu, gQ, tau);
      for (int a = 0; a < 3; ++a) torque[3 * i + a] += electric * tau[a];
      double dm[3] = {-d[0], -d[1], -d[2]};
      tens_t Tm;
      build_tensors(dm, G, &Tm);
      pair_grad_i(qi, mi, Qi, &Tm, gmu, gQ);
      torque_from_grads(mj, Qj, gmu, gQ, tau);
      for (int a = 0; a < 3; ++a) torque[3 * j + a] += electric * tau[a];
    }
  }
  *energy = etot;
  if (virial) memcpy(virial, w, sizeof w);
  return MDO_OK;
}

int mdo_mpole_field_tensor(const mdo_system* s, const mdo_table* t, double alpha,
                           double cutoff, int exclude, double* e) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  const size_t n = s->n;
  memset(e, 0, 3 * n * sizeof(double));
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  tens_t T, Tm;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double d[3];
      const double r2 = pair_d(s, &b, i, j, &d[0], &d[1], &d[2]);
      if (!(r2 <= c2) || excluded(s, exclude, i, j)) continue;
      const double r = sqrt(r2);
      double G[6];
      mdo_ewald_bn(r, alpha, 4, G);
      G[5] = 0;
      build_tensors(d, G, &T);
      double dm[3] = {-d[0], -d[1], -d[2]};
      build_tensors(dm, G, &Tm);
      double Qi[3][3], Qj[3][3];
      quad3(s->quadrupole ? s->quadrupole + 6 * i : zero6, Qi);
      quad3(s->quadrupole ? s->quadrupole + 6 * j : zero6, Qj);
      const double* mi = s->dipole ? s->dipole + 3 * i : zero3v;
      const double* mj = s->dipole ? s->dipole + 3 * j : zero3v;
      /* E_i = -grad phi_j at r_i; phi_j = (q_j - mu_j.d + Q_j:dd) G0(R) */
      for (int a = 0; a < 3; ++a) {
        double v = s->charge[j] * T.t1[a];
        for (int c = 0; c < 3; ++c) v += -mj[c] * T.t2[c * 3 + a];
        for (int c = 0; c < 3; ++c)
          for (int d2 = 0; d2 < 3; ++d2) v += Qj[c][d2] * T.t3[(c * 3 + d2) * 3 + a];
        e[3 * i + a] -= v;
        double w2 = s->charge[i] * Tm.t1[a];
        for (int c = 0; c < 3; ++c) w2 += -mi[c] * Tm.t2[c * 3 + a];
        for (int c = 0; c < 3; ++c)
          for (int d2 = 0; d2 < 3; ++d2) w2 += Qi[c][d2] * Tm.t3[(c * 3 + d2) * 3 + a];
        e[3 * j + a] -= w2;
      }
    }
  }
  return MDO_OK;
}

/* Thole lambda9 (EXTENSION): with lambda3..9 the damped radial functions
 * G_n = B_n - (1 - lambda_{2n+1}) g_n obey dG_n/dR = -R G_{n+1} like the
 * undamped ones, so the generic tensors apply to the damped interaction. */
static double thole_l9(double r, double ai, double aj, double a) {
  const double u = r / cbrt(sqrt(ai * aj));
  const double s1 = a * u * u * u;
  return 1.0 - (1.0 + s1 + (18.0 / 35.0) * s1 * s1 + (9.0 / 35.0) * s1 * s1 * s1) * exp(-s1);
}

int mdo_polar_forces(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                     double thole_a, double electric, int exclude, const double* mu,
                     double* f, double* torque, double* energy, double* virial) {
  int rc = validate_kernel(s, t, cutoff);
  if (rc) return rc;
  const size_t n = s->n;
  memset(f, 0, 3 * n * sizeof(double));
  memset(torque, 0, 3 * n * sizeof(double));
  double w[9] = {0};
  double etot = 0.0;
  const double c2 = cutoff * cutoff;
  box_t b = make_box(s->lx, s->ly, s->lz);
  tens_t T, Tm;
  static const double Z[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double Zq[3][3];
  memcpy(Zq, Z, sizeof Zq);
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double d[3];
      const double r2 = pair_d(s, &b, i, j, &d[0], &d[1], &d[2]);
      if (!(r2 <= c2)) continue;
      if (!(r2 > 0)) return fail(MDO_SINGULARITY, "polar_forces: coincident sites");
      const int excl = excluded(s, exclude, i, j);
      const double r = sqrt(r2);
      double bn[5], g[5], l3, l5, l7;
      mdo_ewald_bn(r, alpha, 4, bn);
      bare_bn(r, 4, g);
      thole_core(r, s->polarizability[i], s->polarizability[j], thole_a, &l3, &l5, &l7);
      const double l9 = thole_l9(r, s->polarizability[i], s->polarizability[j], thole_a);
      double G[6];
      G[0] = 0.0; /* no charge-charge term */
      G[1] = bn[1] - (1.0 - l3) * g[1];
      G[2] = bn[2] - (1.0 - l5) * g[2];
      G[3] = bn[3] - (1.0 - l7) * g[3];
      G[4] = bn[4] - (1.0 - l9) * g[4];
      G[5] = 0.0; /* rank-5 tensors only meet zero quadrupole products */
      build_tensors(d, G, &T);
      double Qi[3][3], Qj[3][3];
      quad3(s->quadrupole ? s->quadrupole + 6 * i : zero6, Qi);
      quad3(s->quadrupole ? s->quadrupole + 6 * j : zero6, Qj);
      const double* di = s->dipole ? s->dipole + 3 * i : zero3v;
      const double* dj = s->dipole ? s->dipole + 3 * j : zero3v;
      const double* ui = mu + 3 * i;
      const double* uj = mu + 3 * j;
      const double qi = excl ? 0.0 : s->charge[i], qj = excl ? 0.0 : s->charge[j];
      /* U = -mu_i.T_ij.mu_j (all pairs) - mu_i.E_{j->i} - mu_j.E_{i->j}
       * (d-scale: not for same-molecule pairs), all in the tensor form */
      double u = pair_energy_tensor(0.0, ui, Zq, 0.0, uj, Zq, &T, 0, 0);
      if (!excl) {
        u += pair_energy_tensor(0.0, ui, Zq, qj, dj, Qj, &T, 0, 0);
        u += pair_energy_tensor(qi, di, Qi, 0.0, uj, Zq, &T, 0, 0);
      }
      etot += electric * u;
      double fi[3];
      for (int e = 0; e < 3; ++e) {
        double du = pair_energy_tensor(0.0, ui, Zq, 0.0, uj, Zq, &T, 1, e);
        if (!excl) {
          du += pair_energy_tensor(0.0, ui, Zq, qj, dj, Qj, &T, 1, e);
          du += pair_energy_tensor(qi, di, Qi, 0.0, uj, Zq, &T, 1, e);
        }
        fi[e] = -electric * du;
        f[3 * i + e] += fi[e];
        f[3 * j + e] -= fi[e];
      }
      add_virial(w, d[0], d[1], d[2], fi[0], fi[1], fi[2]);
      if (excl) continue;
      /* torques on the permanent multipoles in the induced field */
      double gmu[3], gQ[3][3], tau[3];
      pair_grad_i(0.0, uj, Zq, &T, gmu, gQ);
      torque_from_grads(di, Qi, gmu, gQ, tau);
      for (int a = 0; a < 3; ++a) torque[3 * i + a] += electric * tau[a];
      double dm[3] = {-d[0], -d[1], -d[2]};
      build_tensors(dm, G, &Tm);
      pair_grad_i(0.0, ui, Zq, &Tm, gmu, gQ);
      torque_from_grads(dj, Qj, gmu, gQ, tau);
      for (int a = 0; a < 3; ++a) torque[3 * j + a] += electric * tau[a];
    }
  }
  if (energy) *energy = etot;
  if (virial) memcpy(virial, w, sizeof w);
  return MDO_OK;
}

int mdo_pcg(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
            double thole_a, const double* eperm, double tol_debye, size_t max_iter,
            double* mu, size_t* iters, double* last_rms) {
  if (!(tol_debye > 0)) return fail(MDO_CONTRACT, "pcg: tol must be positive");
  if (max_iter < 1) return fail(MDO_CONTRACT, "pcg: max_iter must be >= 1");
  const size_t n = s->n, m = 3 * n;
  double* r = (double*)malloc(m * sizeof(double) + 8);
  double* z = (double*)malloc(m * sizeof(double) + 8);
  double* p = (double*)malloc(m * sizeof(double) + 8);
  double* q = (double*)malloc(m * sizeof(double) + 8);
  double* tp = (double*)malloc(m * sizeof(double) + 8);
  for (size_t i = 0; i < n; ++i) {
    const double pa = s->polarizability[i];
    if (!(pa > 0)) { free(r); free(z); free(p); free(q); free(tp);
      return fail(MDO_CONTRACT, "pcg: polarizabilities must be positive"); }
    for (int a = 0; a < 3; ++a) mu[3 * i + a] = pa * eperm[3 * i + a];
  }
  /* r0 = E - (mu0/alpha - T mu0) = T mu0 */
  int rc = mdo_tmatvec_ewald(s, t, alpha, cutoff, thole_a, mu, r);
  if (rc) { free(r); free(z); free(p); free(q); free(tp); return rc; }
  double rz = 0.0;
  for (size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const size_t k = 3 * i + a;
      r[k] = eperm[k] - (mu[k] / s->polarizability[i] - r[k]);
      z[k] = s->polarizability[i] * r[k];
      p[k] = z[k];
      rz += r[k] * z[k];
    }
  double rms = 0.0;
  for (size_t it = 0; it < max_iter; ++it) {
    rc = mdo_tmatvec_ewald(s, t, alpha, cutoff, thole_a, p, tp);
    if (rc) break;
    double pq = 0.0;
    for (size_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        const size_t k = 3 * i + a;
        q[k] = p[k] / s->polarizability[i] - tp[k];
        pq += p[k] * q[k];
      }
    const double ak = pq != 0.0 ? rz / pq : 0.0;  /* p == 0: r == 0, exact already */
    double dsum = 0.0, rz_new = 0.0;
    for (size_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        const size_t k = 3 * i + a;
        const double dm = ak * p[k];
        mu[k] += dm;
        dsum += dm * dm;
        r[k] -= ak * q[k];
        z[k] = s->polarizability[i] * r[k];
        rz_new += r[k] * z[k];
      }
    rms = sqrt(dsum / (double)n) * MDO_DEBYE;
    *iters = it + 1;
    *last_rms = rms;
    if (rms < tol_debye) break;
    const double bk = rz != 0.0 ? rz_new / rz : 0.0;
    rz = rz_new;
    for (size_t k = 0; k < m; ++k) p[k] = z[k] + bk * p[k];
  }
  free(r); free(z); free(p); free(q); free(tp);
  if (rc) return rc;
  if (!(rms < tol_debye))
    return fail(MDO_CONVERGENCE, "pcg: no convergence after max_iter");
  return MDO_OK;
}
