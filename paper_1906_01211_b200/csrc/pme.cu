// pme.cu -- smooth particle-mesh Ewald, reciprocal space for point charges
// (completes the real-space Ewald of the CHARMM step so its
// energies become physical; the reference is real-space only).
//
// Essmann et al. smooth PME on a K1 x K2 x K3 grid with order-p cardinal
// B-splines: charges spread with FP64 atomics (one thread per site, p^3
// points), cuFFT D2Z, the influence function exp(-pi^2 m^2/a^2)/(pi V m^2)
// times the B-spline moduli (energy and virial reduced per block in a fixed
// order), cuFFT Z2D back to the potential grid, forces gathered per site
// with the spline derivatives. Plus the self energy -a/sqrt(pi) sum q^2 and
// the removal of the excluded (same-molecule) pairs, -q_i q_j erf(a r)/r,
// per site over its molecule partners (deterministic, no atomics).
// Oracle: oracle/ewald_recip.py (direct structure-factor sum).
#include <cufft.h>

#include <cmath>
#include <vector>

#include "common.cuh"

namespace mdg {

constexpr int kMaxOrder = 10;

// theta[j] = M_p(w + j), dtheta[j] = dM_p/du (grid point iu - j)
__device__ __forceinline__ void bspline(double w, int p, double* th, double* dth) {
  double c[kMaxOrder];
  c[0] = w;
  c[1] = 1.0 - w;
  for (int n = 3; n <= p; ++n) {
    if (n == p) {  // derivative from order p-1: dM_p(x) = M_{p-1}(x) - M_{p-1}(x-1)
      dth[0] = c[0];
      for (int j = 1; j < p - 1; ++j) dth[j] = c[j] - c[j - 1];
      dth[p - 1] = -c[p - 2];
    }
    const double inv = 1.0 / (double)(n - 1);
    double prev = 0.0;  // c_{n-1}[j-1]
    for (int j = 0; j < n; ++j) {
      const double cj = (j < n - 1) ? c[j] : 0.0;
      const double x = w + j;
      const double v = (x * cj + ((double)n - x) * prev) * inv;
      prev = cj;
      c[j] = v;
    }
  }
  if (p == 2) {
    dth[0] = 1.0;
    dth[1] = -1.0;
  }
  for (int j = 0; j < p; ++j) th[j] = c[j];
}

struct PmeGeom {
  int k1, k2, k3, p;
  double l1, l2, l3;
};

__device__ __forceinline__ void frac(double x, double L, int K, int& iu, double& w) {
  double u = x / L * (double)K;
  double f = floor(u);
  iu = (int)f;
  w = u - f;
  iu = ((iu % K) + K) % K;
}

__global__ void k_pme_spread(int64_t n, PmeGeom g, const double4* __restrict__ pos,
                             const double4* __restrict__ pq4, double* __restrict__ grid) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double q = pq4[i].z;
  if (q == 0.0) return;
  const double4 r = pos[i];
  int i1, i2, i3;
  double w1, w2, w3;
  frac(r.x, g.l1, g.k1, i1, w1);
  frac(r.y, g.l2, g.k2, i2, w2);
  frac(r.z, g.l3, g.k3, i3, w3);
  double t1[kMaxOrder], t2[kMaxOrder], t3[kMaxOrder], d[kMaxOrder];
  bspline(w1, g.p, t1, d);
  bspline(w2, g.p, t2, d);
  bspline(w3, g.p, t3, d);
  for (int a = 0; a < g.p; ++a) {
    const int x = (i1 - a + g.k1) % g.k1;
    for (int b = 0; b < g.p; ++b) {
      const int y = (i2 - b + g.k2) % g.k2;
      const double qab = q * t1[a] * t2[b];
      double* row = grid + ((size_t)x * g.k2 + y) * g.k3;
      for (int c = 0; c < g.p; ++c) atomicAdd(row + (i3 - c + g.k3) % g.k3, qab * t3[c]);
    }
  }
}

// S(m) *= G(m); energy and virial of the full spectrum (half-spectrum
// entries with 0 < kz < K3/2 stand for two)
__global__ void __launch_bounds__(kBlock) k_pme_convolve(PmeGeom g, double alpha,
                                                        const double* __restrict__ bmod,
                                                        cufftDoubleComplex* __restrict__ s,
                                                        double* __restrict__ partials) {
  const int kzh = g.k3 / 2 + 1;
  const int64_t total = (int64_t)g.k1 * g.k2 * kzh;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  const double V = g.l1 * g.l2 * g.l3;
  const double pa = M_PI * M_PI / (alpha * alpha);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int kz = (int)(e % kzh);
    const int ky = (int)((e / kzh) % g.k2);
    const int kx = (int)(e / ((int64_t)kzh * g.k2));
    const int mx = (kx <= g.k1 / 2) ? kx : kx - g.k1;
    const int my = (ky <= g.k2 / 2) ? ky : ky - g.k2;
    const double m1 = mx / g.l1, m2 = my / g.l2, m3 = kz / g.l3;
    const double msq = m1 * m1 + m2 * m2 + m3 * m3;
    cufftDoubleComplex v = s[e];
    if (msq == 0.0) {
      s[e] = make_cuDoubleComplex(0.0, 0.0);
      continue;
    }
    const double G = exp(-pa * msq) / (M_PI * V * msq) * bmod[kx] * bmod[g.k1 + ky] *
                     bmod[g.k1 + g.k2 + kz];
    const double wz = (kz == 0 || (g.k3 % 2 == 0 && kz == g.k3 / 2)) ? 1.0 : 2.0;
    const double em = 0.5 * wz * G * (v.x * v.x + v.y * v.y);
    const double f = 2.0 * (1.0 + pa * msq) / msq;
    acc[0] += em;
    acc[1] += em * (1.0 - f * m1 * m1);
    acc[2] += em * (-f * m1 * m2);
    acc[3] += em * (-f * m1 * m3);
    acc[4] += em * (1.0 - f * m2 * m2);
    acc[5] += em * (-f * m2 * m3);
    acc[6] += em * (1.0 - f * m3 * m3);
    s[e] = make_cuDoubleComplex(v.x * G, v.y * G);
  }
  block_store_partials<7>(acc, partials);
}

__global__ void k_pme_gather(int64_t n, PmeGeom g, const double4* __restrict__ pos,
                             const double4* __restrict__ pq4, const double* __restrict__ phi,
                             double electric, double4* __restrict__ force) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double q = pq4[i].z;
  double4 f = force[i];
  if (q != 0.0) {
    const double4 r = pos[i];
    int i1, i2, i3;
    double w1, w2, w3;
    frac(r.x, g.l1, g.k1, i1, w1);
    frac(r.y, g.l2, g.k2, i2, w2);
    frac(r.z, g.l3, g.k3, i3, w3);
    double t1[kMaxOrder], t2[kMaxOrder], t3[kMaxOrder], d1[kMaxOrder], d2[kMaxOrder],
        d3[kMaxOrder];
    bspline(w1, g.p, t1, d1);
    bspline(w2, g.p, t2, d2);
    bspline(w3, g.p, t3, d3);
    double gx = 0, gy = 0, gz = 0;
    for (int a = 0; a < g.p; ++a) {
      const int x = (i1 - a + g.k1) % g.k1;
      for (int b = 0; b < g.p; ++b) {
        const int y = (i2 - b + g.k2) % g.k2;
        const double* row = phi + ((size_t)x * g.k2 + y) * g.k3;
        for (int c = 0; c < g.p; ++c) {
          const double ph = __ldg(row + (i3 - c + g.k3) % g.k3);
          gx += d1[a] * t2[b] * t3[c] * ph;
          gy += t1[a] * d2[b] * t3[c] * ph;
          gz += t1[a] * t2[b] * d3[c] * ph;
        }
      }
    }
    const double s = -electric * q;
    f.x += s * gx * g.k1 / g.l1;
    f.y += s * gy * g.k2 / g.l2;
    f.z += s * gz * g.k3 / g.l3;
  }
  force[i] = f;
}

// excluded pairs: -q_i q_j erf(a r)/r for every same-molecule partner j of
// i; i-side force in full, energy / virial halved (each pair seen twice)
__global__ void __launch_bounds__(kBlock) k_pme_excluded(int64_t n, Box b, double alpha,
                                                        double electric,
                                                        const double4* __restrict__ pos,
                                                        const double4* __restrict__ pq4,
                                                        const int32_t* __restrict__ xs,
                                                        const int32_t* __restrict__ xl,
                                                        double4* __restrict__ force,
                                                        double* __restrict__ partials) {
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double4 pi = pos[i];
    const double qi = pq4[i].z;
    double fx = 0, fy = 0, fz = 0;
    for (int32_t k = xs[i]; k < xs[i + 1]; ++k) {
      const int32_t j = xl[k];
      const double4 pj = pos[j];
      double dx, dy, dz;
      const double r2 = min_image(b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
      const double r = sqrt(r2);
      const double qq = electric * qi * pq4[j].z;
      const double er = erf(alpha * r);
      const double dd = (1.1283791670955126 * alpha * exp(-alpha * alpha * r2) - er / r) / r;
      const double s = qq * dd / r;
      acc[0] -= 0.5 * qq * er / r;
      fx += s * dx;
      fy += s * dy;
      fz += s * dz;
      acc[1] += 0.5 * dx * s * dx;
      acc[2] += 0.5 * dx * s * dy;
      acc[3] += 0.5 * dx * s * dz;
      acc[4] += 0.5 * dy * s * dx;
      acc[5] += 0.5 * dy * s * dy;
      acc[6] += 0.5 * dy * s * dz;
      acc[7] += 0.5 * dz * s * dx;
      acc[8] += 0.5 * dz * s * dy;
      acc[9] += 0.5 * dz * s * dz;
    }
    double4 f = force[i];
    f.x += fx;
    f.y += fy;
    f.z += fz;
    force[i] = f;
  }
  block_store_partials<10>(acc, partials);
}

// |b(m)|^2 of the B-spline interpolation (Essmann eq. 4.4), m = 0..K-1
static std::vector<double> bspline_moduli(int K, int p) {
  // M_n at the integers 0..n by the recursion M_n(k) = (k M_{n-1}(k) +
  // (n - k) M_{n-1}(k - 1)) / (n - 1), from M_2(1) = 1
  std::vector<double> M(p + 1, 0.0);
  M[1] = 1.0;
  for (int n = 3; n <= p; ++n) {
    std::vector<double> N(p + 1, 0.0);
    for (int k = 1; k < n; ++k) N[k] = (k * M[k] + (n - k) * M[k - 1]) / (n - 1);
    M = N;
  }
  std::vector<double> out(K);
  for (int j = 0; j < K; ++j) {
    double re = 0, im = 0;
    for (int k = 0; k <= p - 2; ++k) {
      const double arg = 2.0 * M_PI * j * k / K;
      re += M[k + 1] * std::cos(arg);
      im += M[k + 1] * std::sin(arg);
    }
    const double den = re * re + im * im;
    out[j] = den > 1e-12 ? 1.0 / den : 0.0;
  }
  // odd orders vanish at the Nyquist point: the neighbours' mean
  for (int j = 0; j < K; ++j)
    if (out[j] == 0.0) out[j] = 0.5 * (out[(j + K - 1) % K] + out[(j + 1) % K]);
  return out;
}

__global__ void __launch_bounds__(kBlock) k_pme_q2(int64_t n, const double4* __restrict__ pq4,
                                                  double* __restrict__ partials) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[1] = {0.0};
  if (i < n) {
    const double q = pq4[i].z;
    acc[0] = q * q;
  }
  block_store_partials<1>(acc, partials);
}

struct PmeState {
  int k1 = 0, k2 = 0, k3 = 0, p = 0;
  double l1 = 0, l2 = 0, l3 = 0;
  double* grid = nullptr;
  cufftDoubleComplex* spec = nullptr;
  double* bmod = nullptr;
  cufftHandle fwd = 0, inv = 0;
  bool plans = false;
};

void pme_free(mdg_ctx* c) {
  PmeState* s = (PmeState*)c->pme;
  if (!s) return;
  if (s->plans) {
    cufftDestroy(s->fwd);
    cufftDestroy(s->inv);
  }
  cudaFree(s->grid);
  cudaFree(s->spec);
  cudaFree(s->bmod);
  delete s;
  c->pme = nullptr;
}

static void cufft_check(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) throw_error(MDG_CUDA, std::string("cuFFT: ") + what);
}

// results: 80 recip energy, 81..86 virial (xx xy xz yy yz zz), 87 self,
// 88 excluded-pair energy, 89..97 excluded-pair virial (row-major)
void run_pme(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order, double electric,
             bool exclude) {
  PmeState* s = (PmeState*)c->pme;
  if (!s) c->pme = s = new PmeState();
  if (s->k1 != k1 || s->k2 != k2 || s->k3 != k3 || s->p != order || s->l1 != c->lx ||
      s->l2 != c->ly || s->l3 != c->lz) {
    if (s->plans) {
      cufftDestroy(s->fwd);
      cufftDestroy(s->inv);
      s->plans = false;
    }
    cudaFree(s->grid);
    cudaFree(s->spec);
    cudaFree(s->bmod);
    s->grid = nullptr;
    s->spec = nullptr;
    s->bmod = nullptr;
    const size_t nreal = (size_t)k1 * k2 * k3, ncplx = (size_t)k1 * k2 * (k3 / 2 + 1);
    MDG_CUDA_CHECK(cudaMalloc(&s->grid, nreal * sizeof(double)));
    MDG_CUDA_CHECK(cudaMalloc(&s->spec, ncplx * sizeof(cufftDoubleComplex)));
    std::vector<double> bm;
    for (auto [K, L] : {std::pair<int, double>{k1, c->lx}, {k2, c->ly}, {k3, c->lz}}) {
      (void)L;
      auto v = bspline_moduli(K, order);
      bm.insert(bm.end(), v.begin(), v.end());
    }
    MDG_CUDA_CHECK(cudaMalloc(&s->bmod, bm.size() * sizeof(double)));
    MDG_CUDA_CHECK(cudaMemcpy(s->bmod, bm.data(), bm.size() * sizeof(double),
                              cudaMemcpyHostToDevice));
    cufft_check(cufftPlan3d(&s->fwd, k1, k2, k3, CUFFT_D2Z), "plan D2Z");
    cufft_check(cufftPlan3d(&s->inv, k1, k2, k3, CUFFT_Z2D), "plan Z2D");
    s->plans = true;
    s->k1 = k1;
    s->k2 = k2;
    s->k3 = k3;
    s->p = order;
    s->l1 = c->lx;
    s->l2 = c->ly;
    s->l3 = c->lz;
  }
  cufft_check(cufftSetStream(s->fwd, c->stream), "stream");
  cufft_check(cufftSetStream(s->inv, c->stream), "stream");
  const PmeGeom g{k1, k2, k3, order, c->lx, c->ly, c->lz};
  const int64_t n = c->n;
  MDG_CUDA_CHECK(cudaMemsetAsync(s->grid, 0, (size_t)k1 * k2 * k3 * sizeof(double), c->stream));
  MDG_LAUNCH(c, "pme_spread", grid_for(n, 128), 128, 0, k_pme_spread, n, g, c->pos, c->pq4,
             s->grid);
  cufft_check(cufftExecD2Z(s->fwd, s->grid, s->spec), "D2Z");
  const int64_t total = (int64_t)k1 * k2 * (k3 / 2 + 1);
  const int64_t blocks = std::min<int64_t>(grid_for(total), 148 * 32);
  ensure_partials(c, std::max<int64_t>(blocks, grid_for(n)));
  MDG_LAUNCH(c, "pme_convolve", (unsigned)blocks, kBlock, 0, k_pme_convolve, g, alpha, s->bmod,
             s->spec, c->partials);
  finalize_partials(c, blocks, 7, 80, electric);
  cufft_check(cufftExecZ2D(s->inv, s->spec, s->grid), "Z2D");
  MDG_LAUNCH(c, "pme_gather", grid_for(n, 128), 128, 0, k_pme_gather, n, g, c->pos, c->pq4,
             s->grid, electric, c->force);
  MDG_LAUNCH(c, "pme_self", grid_for(n), kBlock, 0, k_pme_q2, n, c->pq4, c->partials);
  finalize_partials(c, grid_for(n), 1, 87, -electric * alpha / std::sqrt(M_PI));
  if (exclude && c->has_mol && c->excl_start) {
    MDG_LAUNCH(c, "pme_excluded", grid_for(n), kBlock, 0, k_pme_excluded, n,
               make_box(c->lx, c->ly, c->lz), alpha, electric, c->pos, c->pq4, c->excl_start,
               c->excl, c->force, c->partials);
    finalize_partials(c, grid_for(n), 10, 88, 1.0);
  }
}

}  // namespace mdg
