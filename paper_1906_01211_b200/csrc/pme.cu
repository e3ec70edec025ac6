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
                                                        double* __restrict__ partials,
                                                        int y0 = 0, int ny = -1) {
  // partials == NULL: the convolution alone (the induced-dipole field).
  // s holds the ky window [y0, y0 + ny) as [k1][ny][k3/2+1] (the whole
  // spectrum when ny < 0; a slab-decomposed part's columns otherwise)
  const int kzh = g.k3 / 2 + 1;
  if (ny < 0) ny = g.k2;
  const int64_t total = (int64_t)g.k1 * ny * kzh;
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  const double V = g.l1 * g.l2 * g.l3;
  const double pa = M_PI * M_PI / (alpha * alpha);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int kz = (int)(e % kzh);
    const int ky = y0 + (int)((e / kzh) % ny);
    const int kx = (int)(e / ((int64_t)kzh * ny));
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
  if (partials) block_store_partials<7>(acc, partials);
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
  // slab decomposition (PcgComm::slab_parts): this domain is part `sl_part`
  // of `sl_parts`; it owns the x-planes [x0, x1) of the real grid and, after
  // the transpose, the ky columns [y0, y1) of the spectrum
  int sl_parts = 0, sl_part = -1;
  cufftHandle pf = 0, pi = 0, px = 0;  // 2D D2Z / Z2D over (y, z); 1D Z2Z along x
  cufftDoubleComplex* sa = nullptr;  // [nx][k2][k3/2+1]: the part's planes
  cufftDoubleComplex* sx = nullptr;  // the same, packed by destination part
  cufftDoubleComplex* sb = nullptr;  // [k1][ny][k3/2+1]: the part's columns
};

static void slab_free(PmeState* s) {
  if (s->sl_parts > 0) {
    cufftDestroy(s->pf);
    cufftDestroy(s->pi);
    if (s->px) cufftDestroy(s->px);
  }
  cudaFree(s->sa);
  cudaFree(s->sx);
  cudaFree(s->sb);
  s->sa = s->sx = s->sb = nullptr;
  s->pf = s->pi = s->px = 0;
  s->sl_parts = 0;
  s->sl_part = -1;
}

static void pme_free_slot(void** slot) {
  PmeState* s = (PmeState*)*slot;
  if (!s) return;
  if (s->plans) {
    cufftDestroy(s->fwd);
    cufftDestroy(s->inv);
  }
  slab_free(s);
  cudaFree(s->grid);
  cudaFree(s->spec);
  cudaFree(s->bmod);
  delete s;
  *slot = nullptr;
}

void pme_free(mdg_ctx* c) {
  pme_free_slot(&c->pme);
  pme_free_slot(&c->pme_pol);
}

static void cufft_check(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) throw_error(MDG_CUDA, std::string("cuFFT: ") + what);
}

// results: 80 recip energy, 81..86 virial (xx xy xz yy yz zz), 87 self,
// 88 excluded-pair energy, 89..97 excluded-pair virial (row-major)
static PmeState* pme_state(mdg_ctx* c, void** slot, int k1, int k2, int k3, int order) {
  PmeState* s = (PmeState*)*slot;
  if (!s) *slot = s = new PmeState();
  if (s->k1 != k1 || s->k2 != k2 || s->k3 != k3 || s->p != order || s->l1 != c->lx ||
      s->l2 != c->ly || s->l3 != c->lz) {
    if (s->plans) {
      cufftDestroy(s->fwd);
      cufftDestroy(s->inv);
      s->plans = false;
    }
    slab_free(s);
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
  return s;
}

void pme_setup(mdg_ctx* c, int k1, int k2, int k3, int order) {
  pme_state(c, &c->pme, k1, k2, k3, order);
}

void run_pme(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order, double electric,
             bool exclude) {
  pme_setup(c, k1, k2, k3, order);
  PmeState* s = (PmeState*)c->pme;
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


// ---- permanent multipoles (q, mu, Theta) --------------------------------------
// Site operator M = q + mu.grad + Q:grad grad (the real-space kernels'
// convention, Q = Theta/3): the grid holds sum_j M_j(grad_j) W_j(k) with
// W_j(k) = prod_a M_p(u_ja - k_a) and grad_a = (K_a/L_a) d/du_a; after the
// convolution the potential phi and its derivatives to third order are
// gathered at every site: E = 1/2 sum M_i phi_i (from the convolution),
// F_i = -M_i grad phi_i, tau_i = grad phi_i x mu_i + 2 (Q G - G Q)_{zy,xz,yx}
// with G = grad grad phi_i. Self energy and the excluded (same-molecule)
// pairs' erf-kernel interaction complete the Ewald sum.
// Oracle: oracle/ewald_mpole.py (direct structure-factor sum).

// th[d][j] = d-th derivative of M_p at w + j (grid point iu - j), d = 0..3
__device__ __forceinline__ void bspline_d3(double w, int p, double (*th)[kMaxOrder]) {
  double c[kMaxOrder];         // M_n(w + j), built up n = 2..p
  double lo[4][kMaxOrder];     // M_{p-3}, M_{p-2}, M_{p-1}, M_p
  c[0] = w;
  c[1] = 1.0 - w;
  for (int j = 2; j < kMaxOrder; ++j) c[j] = 0.0;
  auto save = [&](int n) {
    const int k = n - (p - 3);
    if (k >= 0 && k < 4)
      for (int j = 0; j < kMaxOrder; ++j) lo[k][j] = (j < n) ? c[j] : 0.0;
  };
  save(2);
  for (int n = 3; n <= p; ++n) {
    const double inv = 1.0 / (double)(n - 1);
    double prev = 0.0;
    for (int j = 0; j < n; ++j) {
      const double cj = (j < n - 1) ? c[j] : 0.0;
      const double x = w + j;
      const double v = (x * cj + ((double)n - x) * prev) * inv;
      prev = cj;
      c[j] = v;
    }
    save(n);
  }
  // M^(d)(x) = sum_l (-1)^l C(d, l) M_{p-d}(x - l)
  const double bin[4][4] = {{1, 0, 0, 0}, {1, -1, 0, 0}, {1, -2, 1, 0}, {1, -3, 3, -1}};
  for (int d = 0; d < 4; ++d)
    for (int j = 0; j < p; ++j) {
      double v = 0.0;
      for (int l = 0; l <= d; ++l)
        if (j - l >= 0) v += bin[d][l] * lo[3 - d][j - l];
      th[d][j] = v;
    }
}

__global__ void k_pme_spread_mp(int64_t n, PmeGeom g, const double4* __restrict__ pos,
                                const double4* __restrict__ pq4, const double4* __restrict__ mp,
                                double* __restrict__ grid, const double4* __restrict__ ind) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 r = pos[i];
  const double q = pq4[i].z;
  double4 m0 = mp[3 * i];
  const double4 m1 = mp[3 * i + 1];
  if (ind) {  // + induced dipoles (the polarization forces' combined set)
    const double4 u = ind[i];
    m0.x += u.x;
    m0.y += u.y;
    m0.z += u.z;
  }
  const double qzz = mp[3 * i + 2].x;
  const double s1 = g.k1 / g.l1, s2 = g.k2 / g.l2, s3 = g.k3 / g.l3;
  // operator coefficients in fractional derivatives
  const double d1 = m0.x * s1, d2 = m0.y * s2, d3 = m0.z * s3;
  const double q11 = m0.w * s1 * s1, q22 = m1.z * s2 * s2, q33 = qzz * s3 * s3;
  const double q12 = 2.0 * m1.x * s1 * s2, q13 = 2.0 * m1.y * s1 * s3, q23 = 2.0 * m1.w * s2 * s3;
  int i1, i2, i3;
  double w1, w2, w3;
  frac(r.x, g.l1, g.k1, i1, w1);
  frac(r.y, g.l2, g.k2, i2, w2);
  frac(r.z, g.l3, g.k3, i3, w3);
  double a[4][kMaxOrder], b[4][kMaxOrder], t[4][kMaxOrder];
  bspline_d3(w1, g.p, a);
  bspline_d3(w2, g.p, b);
  bspline_d3(w3, g.p, t);
  for (int ia = 0; ia < g.p; ++ia) {
    const int x = (i1 - ia + g.k1) % g.k1;
    for (int ib = 0; ib < g.p; ++ib) {
      const int y = (i2 - ib + g.k2) % g.k2;
      // terms by the z-derivative order they multiply
      const double c0 = q * a[0][ia] * b[0][ib] + d1 * a[1][ia] * b[0][ib] +
                        d2 * a[0][ia] * b[1][ib] + q11 * a[2][ia] * b[0][ib] +
                        q22 * a[0][ia] * b[2][ib] + q12 * a[1][ia] * b[1][ib];
      const double c1 = d3 * a[0][ia] * b[0][ib] + q13 * a[1][ia] * b[0][ib] +
                        q23 * a[0][ia] * b[1][ib];
      const double c2 = q33 * a[0][ia] * b[0][ib];
      double* row = grid + ((size_t)x * g.k2 + y) * g.k3;
      for (int ic = 0; ic < g.p; ++ic)
        atomicAdd(row + (i3 - ic + g.k3) % g.k3, c0 * t[0][ic] + c1 * t[1][ic] + c2 * t[2][ic]);
    }
  }
}

// phi derivatives at each site -> forces, torques (accumulated); partials:
// 0 energy 1/2 sum M_i phi_i (check of the convolution energy)
__global__ void __launch_bounds__(kBlock) k_pme_gather_mp(int64_t n, PmeGeom g,
                                                         const double4* __restrict__ pos,
                                                         const double4* __restrict__ pq4,
                                                         const double4* __restrict__ mp,
                                                         const double* __restrict__ phi,
                                                         double electric,
                                                         double4* __restrict__ force,
                                                         double4* __restrict__ torque,
                                                         double* __restrict__ partials,
                                                         const double4* __restrict__ ind,
                                                         int write_forces) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[1] = {0.0};
  if (i < n) {
    const double4 r = pos[i];
    int i1, i2, i3;
    double w1, w2, w3;
    frac(r.x, g.l1, g.k1, i1, w1);
    frac(r.y, g.l2, g.k2, i2, w2);
    frac(r.z, g.l3, g.k3, i3, w3);
    double a[4][kMaxOrder], b[4][kMaxOrder], t[4][kMaxOrder];
    bspline_d3(w1, g.p, a);
    bspline_d3(w2, g.p, b);
    bspline_d3(w3, g.p, t);
    // fractional derivatives: f[dx][dy][dz] for dx + dy + dz <= 3
    double f0 = 0, fx = 0, fy = 0, fz = 0, fxx = 0, fyy = 0, fzz = 0, fxy = 0, fxz = 0, fyz = 0;
    double fxxx = 0, fyyy = 0, fzzz = 0, fxxy = 0, fxxz = 0, fxyy = 0, fyyz = 0, fxzz = 0,
           fyzz = 0, fxyz = 0;
    for (int ia = 0; ia < g.p; ++ia) {
      const int x = (i1 - ia + g.k1) % g.k1;
      for (int ib = 0; ib < g.p; ++ib) {
        const int y = (i2 - ib + g.k2) % g.k2;
        const double* row = phi + ((size_t)x * g.k2 + y) * g.k3;
        double z0 = 0, z1 = 0, z2 = 0, z3 = 0;  // sums over z with t0..t3
        for (int ic = 0; ic < g.p; ++ic) {
          const double ph = __ldg(row + (i3 - ic + g.k3) % g.k3);
          z0 += t[0][ic] * ph;
          z1 += t[1][ic] * ph;
          z2 += t[2][ic] * ph;
          z3 += t[3][ic] * ph;
        }
        const double a0 = a[0][ia], a1 = a[1][ia], a2 = a[2][ia], a3 = a[3][ia];
        const double b0 = b[0][ib], b1 = b[1][ib], b2 = b[2][ib], b3 = b[3][ib];
        f0 += a0 * b0 * z0;
        fx += a1 * b0 * z0;
        fy += a0 * b1 * z0;
        fz += a0 * b0 * z1;
        fxx += a2 * b0 * z0;
        fyy += a0 * b2 * z0;
        fzz += a0 * b0 * z2;
        fxy += a1 * b1 * z0;
        fxz += a1 * b0 * z1;
        fyz += a0 * b1 * z1;
        fxxx += a3 * b0 * z0;
        fyyy += a0 * b3 * z0;
        fzzz += a0 * b0 * z3;
        fxxy += a2 * b1 * z0;
        fxxz += a2 * b0 * z1;
        fxyy += a1 * b2 * z0;
        fyyz += a0 * b2 * z1;
        fxzz += a1 * b0 * z2;
        fyzz += a0 * b1 * z2;
        fxyz += a1 * b1 * z1;
      }
    }
    const double s1 = g.k1 / g.l1, s2 = g.k2 / g.l2, s3 = g.k3 / g.l3;
    // Cartesian gradient G1, Hessian G2, third derivatives G3
    const double g1x = s1 * fx, g1y = s2 * fy, g1z = s3 * fz;
    const double hxx = s1 * s1 * fxx, hyy = s2 * s2 * fyy, hzz = s3 * s3 * fzz;
    const double hxy = s1 * s2 * fxy, hxz = s1 * s3 * fxz, hyz = s2 * s3 * fyz;
    const double txxx = s1 * s1 * s1 * fxxx, tyyy = s2 * s2 * s2 * fyyy, tzzz = s3 * s3 * s3 * fzzz;
    const double txxy = s1 * s1 * s2 * fxxy, txxz = s1 * s1 * s3 * fxxz;
    const double txyy = s1 * s2 * s2 * fxyy, tyyz = s2 * s2 * s3 * fyyz;
    const double txzz = s1 * s3 * s3 * fxzz, tyzz = s2 * s3 * s3 * fyzz;
    const double txyz = s1 * s2 * s3 * fxyz;
    const double q = pq4[i].z;
    const double4 m0 = mp[3 * i], m1 = mp[3 * i + 1];
    // forces act on the whole dipole (permanent + induced); torques only on
    // the permanent one (induced dipoles are not attached to the frame)
    const double4 u = ind ? ind[i] : make_double4(0.0, 0.0, 0.0, 0.0);
    const double dx = m0.x + u.x, dy = m0.y + u.y, dz = m0.z + u.z;
    const double px = m0.x, py = m0.y, pz = m0.z;
    const double Qxx = m0.w, Qxy = m1.x, Qxz = m1.y, Qyy = m1.z, Qyz = m1.w,
                 Qzz = mp[3 * i + 2].x;
    acc[0] = 0.5 * electric *
             (q * f0 + dx * g1x + dy * g1y + dz * g1z + Qxx * hxx + Qyy * hyy + Qzz * hzz +
              2.0 * (Qxy * hxy + Qxz * hxz + Qyz * hyz));
    // F_a = -(q g1_a + sum_b H_ab d_b + sum_bc Q_bc T_abc)
    const double Fx = q * g1x + hxx * dx + hxy * dy + hxz * dz + Qxx * txxx + Qyy * txyy +
                      Qzz * txzz + 2.0 * (Qxy * txxy + Qxz * txxz + Qyz * txyz);
    const double Fy = q * g1y + hxy * dx + hyy * dy + hyz * dz + Qxx * txxy + Qyy * tyyy +
                      Qzz * tyzz + 2.0 * (Qxy * txyy + Qxz * txyz + Qyz * tyyz);
    const double Fz = q * g1z + hxz * dx + hyz * dy + hzz * dz + Qxx * txxz + Qyy * tyyz +
                      Qzz * tzzz + 2.0 * (Qxy * txyz + Qxz * txzz + Qyz * tyzz);
    if (write_forces) {
      double4 f = force[i];
      f.x -= electric * Fx;
      f.y -= electric * Fy;
      f.z -= electric * Fz;
      force[i] = f;
    }
    // tau = grad phi x mu + 2 (M_zy, M_xz, M_yx), M = Q H - H Q
    double tx = g1y * pz - g1z * py, ty = g1z * px - g1x * pz, tz = g1x * py - g1y * px;
    const double Mzy = (Qxz * hxy + Qyz * hyy + Qzz * hyz) - (hxz * Qxy + hyz * Qyy + hzz * Qyz);
    const double Mxz = (Qxx * hxz + Qxy * hyz + Qxz * hzz) - (hxx * Qxz + hxy * Qyz + hxz * Qzz);
    const double Myx = (Qxy * hxx + Qyy * hxy + Qyz * hxz) - (hxy * Qxx + hyy * Qxy + hyz * Qxz);
    tx += 2.0 * Mzy;
    ty += 2.0 * Mxz;
    tz += 2.0 * Myx;
    if (write_forces) {
      double4 tq = torque[i];
      tq.x += electric * tx;
      tq.y += electric * ty;
      tq.z += electric * tz;
      torque[i] = tq;
    }
  }
  block_store_partials<1>(acc, partials);
}

// partials: 0 sum q^2, 1 sum |mu|^2, 2 sum Q:Q
__global__ void __launch_bounds__(kBlock) k_pme_self_mp(int64_t n, const double4* __restrict__ pq4,
                                                       const double4* __restrict__ mp,
                                                       double* __restrict__ partials) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[3] = {0, 0, 0};
  if (i < n) {
    const double q = pq4[i].z;
    const double4 m0 = mp[3 * i], m1 = mp[3 * i + 1];
    const double zz = mp[3 * i + 2].x;
    acc[0] = q * q;
    acc[1] = m0.x * m0.x + m0.y * m0.y + m0.z * m0.z;
    acc[2] = m0.w * m0.w + m1.z * m1.z + zz * zz +
             2.0 * (m1.x * m1.x + m1.y * m1.y + m1.w * m1.w);
  }
  block_store_partials<3>(acc, partials);
}

// One multipole pair (i-side), the real-space kernels' closed form
// (csrc/mpole.cu) with radial functions G[0..5]: energy U, g = dU/dR,
// gm = dU/dd_i, GQ = dU/dQ_i (xx, xy, xz, yy, yz, zz).
struct MpSite {
  double q, dx, dy, dz, Q[6];
};

__device__ __forceinline__ double mp_pair(const MpSite& a, const MpSite& b, const double* G,
                                          double x, double y, double z, double* g, double* gm,
                                          double* GQ) {
  auto qv = [](const double* Q, double u, double v, double w, double& ox, double& oy,
               double& oz) {
    ox = Q[0] * u + Q[1] * v + Q[2] * w;
    oy = Q[1] * u + Q[3] * v + Q[4] * w;
    oz = Q[2] * u + Q[4] * v + Q[5] * w;
  };
  const double qi = a.q, dix = a.dx, diy = a.dy, diz = a.dz;
  const double qj = b.q, djx = b.dx, djy = b.dy, djz = b.dz;
  const double* Qi = a.Q;
  const double* Qj = b.Q;
  double vix, viy, viz, vjx, vjy, vjz;
  qv(Qi, x, y, z, vix, viy, viz);
  qv(Qj, x, y, z, vjx, vjy, vjz);
  const double dir = dix * x + diy * y + diz * z, djr = djx * x + djy * y + djz * z;
  const double qir = x * vix + y * viy + z * viz, qjr = x * vjx + y * vjy + z * vjz;
  const double dij = dix * djx + diy * djy + diz * djz;
  const double diqj = dix * vjx + diy * vjy + diz * vjz;
  const double djqi = djx * vix + djy * viy + djz * viz;
  const double qiqj = Qi[0] * Qj[0] + Qi[3] * Qj[3] + Qi[5] * Qj[5] +
                      2.0 * (Qi[1] * Qj[1] + Qi[2] * Qj[2] + Qi[4] * Qj[4]);
  const double qvv = vix * vjx + viy * vjy + viz * vjz;
  const double C0 = qi * qj, C1 = qi * djr - qj * dir + dij;
  const double C2 = qi * qjr + qj * qir - dir * djr + 2.0 * (diqj - djqi + qiqj);
  const double C3 = -dir * qjr + qir * djr - 4.0 * qvv, C4 = qir * qjr;
  double a1x, a1y, a1z, a2x, a2y, a2z, b1x, b1y, b1z, b2x, b2y, b2z;
  qv(Qj, dix, diy, diz, a1x, a1y, a1z);
  qv(Qi, djx, djy, djz, a2x, a2y, a2z);
  qv(Qi, vjx, vjy, vjz, b1x, b1y, b1z);
  qv(Qj, vix, viy, viz, b2x, b2y, b2z);
  const double s = C0 * G[1] + C1 * G[2] + C2 * G[3] + C3 * G[4] + C4 * G[5];
  g[0] = G[1] * (qi * djx - qj * dix) +
         G[2] * (2.0 * (qi * vjx + qj * vix) - djr * dix - dir * djx + 2.0 * (a1x - a2x)) +
         G[3] * (-qjr * dix - 2.0 * dir * vjx + 2.0 * djr * vix + qir * djx - 4.0 * (b1x + b2x)) +
         G[4] * 2.0 * (qjr * vix + qir * vjx) - s * x;
  g[1] = G[1] * (qi * djy - qj * diy) +
         G[2] * (2.0 * (qi * vjy + qj * viy) - djr * diy - dir * djy + 2.0 * (a1y - a2y)) +
         G[3] * (-qjr * diy - 2.0 * dir * vjy + 2.0 * djr * viy + qir * djy - 4.0 * (b1y + b2y)) +
         G[4] * 2.0 * (qjr * viy + qir * vjy) - s * y;
  g[2] = G[1] * (qi * djz - qj * diz) +
         G[2] * (2.0 * (qi * vjz + qj * viz) - djr * diz - dir * djz + 2.0 * (a1z - a2z)) +
         G[3] * (-qjr * diz - 2.0 * dir * vjz + 2.0 * djr * viz + qir * djz - 4.0 * (b1z + b2z)) +
         G[4] * 2.0 * (qjr * viz + qir * vjz) - s * z;
  const double c1 = G[1] * qj + G[2] * djr + G[3] * qjr;
  gm[0] = G[1] * djx + 2.0 * G[2] * vjx - c1 * x;
  gm[1] = G[1] * djy + 2.0 * G[2] * vjy - c1 * y;
  gm[2] = G[1] * djz + 2.0 * G[2] * vjz - c1 * z;
  const double crr = G[2] * qj + G[3] * djr + G[4] * qjr, g2 = 2.0 * G[2], g3 = 2.0 * G[3];
  GQ[0] = crr * x * x - G[2] * (2.0 * djx * x) + g2 * Qj[0] - g3 * (2.0 * x * vjx);
  GQ[3] = crr * y * y - G[2] * (2.0 * djy * y) + g2 * Qj[3] - g3 * (2.0 * y * vjy);
  GQ[5] = crr * z * z - G[2] * (2.0 * djz * z) + g2 * Qj[5] - g3 * (2.0 * z * vjz);
  GQ[1] = crr * x * y - G[2] * (djx * y + x * djy) + g2 * Qj[1] - g3 * (x * vjy + vjx * y);
  GQ[2] = crr * x * z - G[2] * (djx * z + x * djz) + g2 * Qj[2] - g3 * (x * vjz + vjx * z);
  GQ[4] = crr * y * z - G[2] * (djy * z + y * djz) + g2 * Qj[4] - g3 * (y * vjz + vjy * z);
  return C0 * G[0] + C1 * G[1] + C2 * G[2] + C3 * G[3] + C4 * G[4];
}

__device__ __forceinline__ MpSite mp_site(const double4* mp, const double4* pq4, int64_t i,
                                          const double4* ind) {
  const double4 m0 = mp[3 * i], m1 = mp[3 * i + 1];
  const double4 u = ind ? ind[i] : make_double4(0.0, 0.0, 0.0, 0.0);
  return MpSite{pq4[i].z, m0.x + u.x, m0.y + u.y, m0.z + u.z,
                {m0.w, m1.x, m1.y, m1.z, m1.w, mp[3 * i + 2].x}};
}

// Excluded (same-molecule) pairs: remove their erf(a r)/r-kernel multipole
// interaction (B_n = bare - erfc). One thread per site over its partners:
// i-side force and torque in full, energy halved (each pair seen twice).
// With induced dipoles (ind != NULL, the polarization forces): the combined
// set's interaction minus the induced-induced part (mutual induction keeps
// every pair in real space), torques on the permanent multipoles only.
__global__ void __launch_bounds__(kBlock) k_pme_excluded_mp(int64_t n, Box bx, double alpha,
                                                           double electric,
                                                           const double4* __restrict__ pos,
                                                           const double4* __restrict__ pq4,
                                                           const double4* __restrict__ mp,
                                                           const int32_t* __restrict__ xs,
                                                           const int32_t* __restrict__ xl,
                                                           double4* __restrict__ force,
                                                           double4* __restrict__ torque,
                                                           double* __restrict__ partials,
                                                           const double4* __restrict__ ind,
                                                           int write_forces) {
  double acc[1] = {0.0};
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double4 pi = pos[i];
    const MpSite si = mp_site(mp, pq4, i, ind);
    const double4 m0i = mp[3 * i];
    double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
    for (int32_t k = xs[i]; k < xs[i + 1]; ++k) {
      const int32_t j = xl[k];
      const double4 pj = pos[j];
      double x, y, z;
      const double r2 = min_image(bx, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, x, y, z);
      const double r = sqrt(r2);
      const double inv_r = 1.0 / r, inv_r2 = inv_r * inv_r;
      double G[6];
      ewald_bn<5>(r, inv_r, inv_r2, alpha, G);
      double bare = inv_r;
      for (int q = 0; q < 6; ++q) {
        if (q > 0) bare *= (double)(2 * q - 1) * inv_r2;
        G[q] = electric * (bare - G[q]);  // erf kernel
      }
      const MpSite sj = mp_site(mp, pq4, j, ind);
      double g[3], gm[3], GQ[6];
      const double u = mp_pair(si, sj, G, x, y, z, g, gm, GQ);
      acc[0] -= 0.5 * u;
      // removing the pair: F_i += dU/dR (the pair force on i is -dU/dR)
      fx += g[0];
      fy += g[1];
      fz += g[2];
      if (ind) {  // keep the induced-induced part
        const double4 ui = ind[i], uj = ind[j];
        const MpSite a{0.0, ui.x, ui.y, ui.z, {0, 0, 0, 0, 0, 0}};
        const MpSite b{0.0, uj.x, uj.y, uj.z, {0, 0, 0, 0, 0, 0}};
        double h[3], hm[3], HQ[6];
        mp_pair(a, b, G, x, y, z, h, hm, HQ);
        fx -= h[0];
        fy -= h[1];
        fz -= h[2];
      }
      // torque on the permanent multipoles of i: gm x d_perm + quadrupole term
      double ux = gm[1] * m0i.z - gm[2] * m0i.y, uy = gm[2] * m0i.x - gm[0] * m0i.z,
             uz = gm[0] * m0i.y - gm[1] * m0i.x;
      const double* Qi = si.Q;
      const double Mzy = (Qi[2] * GQ[1] + Qi[4] * GQ[3] + Qi[5] * GQ[4]) -
                         (GQ[2] * Qi[1] + GQ[4] * Qi[3] + GQ[5] * Qi[4]);
      const double Mxz = (Qi[0] * GQ[2] + Qi[1] * GQ[4] + Qi[2] * GQ[5]) -
                         (GQ[0] * Qi[2] + GQ[1] * Qi[4] + GQ[2] * Qi[5]);
      const double Myx = (Qi[1] * GQ[0] + Qi[3] * GQ[1] + Qi[4] * GQ[2]) -
                         (GQ[1] * Qi[0] + GQ[3] * Qi[1] + GQ[4] * Qi[2]);
      ux += 2.0 * Mzy;
      uy += 2.0 * Mxz;
      uz += 2.0 * Myx;
      tx -= ux;
      ty -= uy;
      tz -= uz;
    }
    if (write_forces) {
      double4 f = force[i];
      f.x += fx;
      f.y += fy;
      f.z += fz;
      force[i] = f;
      double4 t = torque[i];
      t.x += tx;
      t.y += ty;
      t.z += tz;
      torque[i] = t;
    }
  }
  block_store_partials<1>(acc, partials);
}

// results: 80 recip energy (convolution), 88 excluded, 98 recip energy from
// the gathered potentials (check), 104-106 sums of q^2, |mu|^2, Q:Q for the
// self energy (formed on the host); force / torque ADDED to
// ---- replicated-grid reciprocal space over the domains of a group ----------
// Each domain spreads its owned sites into its own grid; the grids are
// summed (comm->grid_sum: on one device into the first domain's grid, which
// every domain then reads; across NCCL ranks an in-place all-reduce of each
// rank's grid); the summed grid is transformed once per device; every
// domain gathers its owned sites from it. The energy of the convolution is
// taken on one domain (comm->recip_root); self and excluded-pair terms are
// per owned site. A single domain is the case comm == NULL.
struct PmeDoms {
  std::vector<mdg_ctx*> doms;
  std::vector<PmeState*> st;
  PcgComm* comm;
  bool shared;  // one device: the first domain's grid serves all
  PmeGeom g;
  size_t count;

  // slab decomposition: P parts, part p owns x-planes [x0[p], x0[p+1]) of
  // the real grid and ky columns [y0[p], y0[p+1]) of the spectrum; kzh =
  // k3/2+1 complex per (x, y) line
  int P = 0;
  std::vector<int> x0, y0;
  int64_t kzh = 0;

  PmeDoms(const std::vector<mdg_ctx*>& d, PcgComm* cm, bool pol, int k1, int k2, int k3,
          int order)
      : doms(d), comm(cm) {
    for (mdg_ctx* c : doms)
      st.push_back(pme_state(c, pol ? &c->pme_pol : &c->pme, k1, k2, k3, order));
    mdg_ctx* c0 = doms[0];
    g = PmeGeom{k1, k2, k3, order, c0->lx, c0->ly, c0->lz};
    count = (size_t)k1 * k2 * k3;
    shared = comm && comm->grid_shared();
    P = comm ? comm->slab_parts() : 0;
    if (P > 0) slab_setup();
  }
  int part(size_t k) const { return comm->slab_part((int)k); }
  int64_t nx(int p) const { return x0[p + 1] - x0[p]; }
  int64_t ny(int p) const { return y0[p + 1] - y0[p]; }
  void slab_setup() {
    if (g.k1 < P || g.k2 < P)
      throw_error(MDG_CONTRACT, "pme: slab decomposition needs K1, K2 >= the number of parts");
    kzh = g.k3 / 2 + 1;
    for (int p = 0; p <= P; ++p) {
      x0.push_back((int)((int64_t)p * g.k1 / P));
      y0.push_back((int)((int64_t)p * g.k2 / P));
    }
    for (size_t k = 0; k < doms.size(); ++k) {
      PmeState* s = st[k];
      const int p = part(k);
      mdg_ctx* c = doms[k];
      if (s->sl_parts != P || s->sl_part != p) {
        slab_free(s);
        const size_t na = (size_t)nx(p) * g.k2 * kzh, nb = (size_t)g.k1 * ny(p) * kzh;
        MDG_CUDA_CHECK(cudaMalloc(&s->sa, na * sizeof(cufftDoubleComplex)));
        MDG_CUDA_CHECK(cudaMalloc(&s->sx, na * sizeof(cufftDoubleComplex)));
        MDG_CUDA_CHECK(cudaMalloc(&s->sb, nb * sizeof(cufftDoubleComplex)));
        int n2[2] = {g.k2, g.k3};
        cufft_check(cufftPlanMany(&s->pf, 2, n2, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z,
                                  (int)nx(p)),
                    "plan slab D2Z");
        cufft_check(cufftPlanMany(&s->pi, 2, n2, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D,
                                  (int)nx(p)),
                    "plan slab Z2D");
        // along x over the part's columns: element (x, col) at x * B + col
        int n1[1] = {g.k1};
        const int B = (int)(ny(p) * kzh);
        cufft_check(cufftPlanMany(&s->px, 1, n1, n1, B, 1, n1, B, 1, CUFFT_Z2Z, B),
                    "plan slab x");
        s->sl_parts = P;
        s->sl_part = p;
      }
      cufft_check(cufftSetStream(s->pf, c->stream), "stream");
      cufft_check(cufftSetStream(s->pi, c->stream), "stream");
      cufft_check(cufftSetStream(s->px, c->stream), "stream");
    }
  }
  // offsets of the transposes: forward, part p's packed planes go to part q
  // (block [nx_p][ny_q][kzh] at nx_p * y0[q] * kzh in p's send buffer) and
  // land as rows x0[p].. of q's column buffer
  void slab_offsets(std::vector<int64_t>& soff, std::vector<int64_t>& doff,
                    std::vector<int64_t>& cnt, std::vector<int64_t>& cntT) const {
    soff.assign(P * P, 0);
    doff.assign(P * P, 0);
    cnt.assign(P * P, 0);
    cntT.assign(P * P, 0);
    for (int p = 0; p < P; ++p)
      for (int q = 0; q < P; ++q) {
        soff[p * P + q] = nx(p) * y0[q] * kzh;
        cnt[p * P + q] = nx(p) * ny(q) * kzh;
        doff[q * P + p] = (int64_t)x0[p] * ny(q) * kzh;
        cntT[q * P + p] = cnt[p * P + q];
      }
  }
  void slab_solve(double alpha, double electric, int slot) {
    std::vector<double*> grids;
    std::vector<cufftDoubleComplex*> sx, sb;
    for (PmeState* s : st) {
      grids.push_back(s->grid);
      sx.push_back(s->sx);
      sb.push_back(s->sb);
    }
    const int n = (int)doms.size();
    const int64_t plane = (int64_t)g.k2 * g.k3;
    std::vector<int64_t> off(P + 1);
    for (int p = 0; p <= P; ++p) off[p] = x0[p] * plane;
    comm->slab_reduce(grids.data(), n, off.data());
    std::vector<int64_t> soff, doff, cnt, cntT;
    slab_offsets(soff, doff, cnt, cntT);
    const size_t z = sizeof(cufftDoubleComplex);
    // 2D transforms of the part's planes, packed by destination part
    for (int k = 0; k < n; ++k) {
      PmeState* s = st[k];
      const int p = part(k);
      cufft_check(cufftExecD2Z(s->pf, s->grid + off[p], s->sa), "slab D2Z");
      for (int q = 0; q < P; ++q)
        if (nx(p) && ny(q))
          MDG_CUDA_CHECK(cudaMemcpy2DAsync(s->sx + soff[p * P + q], ny(q) * kzh * z,
                                           s->sa + y0[q] * kzh, g.k2 * kzh * z, ny(q) * kzh * z,
                                           nx(p), cudaMemcpyDeviceToDevice, doms[k]->stream));
    }
    comm->slab_alltoall(sx.data(), sb.data(), n, soff.data(), doff.data(), cnt.data());
    // along x, convolution on the part's columns (its energy share into
    // `slot`: the domains' slots are summed), back along x
    for (int k = 0; k < n; ++k) {
      mdg_ctx* c = doms[k];
      PmeState* s = st[k];
      const int p = part(k);
      cufft_check(cufftExecZ2Z(s->px, s->sb, s->sb, CUFFT_FORWARD), "slab x fwd");
      const int64_t total = (int64_t)g.k1 * ny(p) * kzh;
      const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(grid_for(total), 148 * 32));
      const bool energy = slot >= 0;
      if (energy) ensure_partials(c, blocks);
      MDG_LAUNCH(c, "pme_convolve", (unsigned)blocks, kBlock, 0, k_pme_convolve, g, alpha,
                 s->bmod, s->sb, energy ? c->partials : (double*)nullptr, y0[p], (int)ny(p));
      if (energy) finalize_partials(c, blocks, 1, slot, electric);
      cufft_check(cufftExecZ2Z(s->px, s->sb, s->sb, CUFFT_INVERSE), "slab x inv");
    }
    comm->slab_alltoall(sb.data(), sx.data(), n, doff.data(), soff.data(), cntT.data());
    for (int k = 0; k < n; ++k) {
      PmeState* s = st[k];
      const int p = part(k);
      for (int q = 0; q < P; ++q)
        if (nx(p) && ny(q))
          MDG_CUDA_CHECK(cudaMemcpy2DAsync(s->sa + y0[q] * kzh, g.k2 * kzh * z,
                                           s->sx + soff[p * P + q], ny(q) * kzh * z,
                                           ny(q) * kzh * z, nx(p), cudaMemcpyDeviceToDevice,
                                           doms[k]->stream));
      cufft_check(cufftExecZ2D(s->pi, s->sa, s->grid + off[p]), "slab Z2D");
    }
    comm->slab_allgather(grids.data(), n, off.data());
  }
  void clear(size_t k) {
    MDG_CUDA_CHECK(cudaMemsetAsync(st[k]->grid, 0, count * sizeof(double), doms[k]->stream));
  }
  void sum() {
    if (!comm || P > 0) return;  // slab: reduced onto the parts in slab_solve
    std::vector<double*> grids;
    for (PmeState* s : st) grids.push_back(s->grid);
    comm->grid_sum(grids.data(), (int)grids.size(), count);
  }
  // the domains that transform (one per device)
  bool solves(size_t k) const { return !shared || k == 0; }
  bool root(size_t k) const { return comm ? comm->recip_root((int)k) : k == 0; }
  const double* phi(size_t k) const { return shared ? st[0]->grid : st[k]->grid; }
  // forward FFT, convolution (energy into `slot` of the root when >= 0),
  // inverse FFT
  void solve(double alpha, double electric, int slot) {
    if (P > 0) return slab_solve(alpha, electric, slot);
    const int64_t total = (int64_t)g.k1 * g.k2 * (g.k3 / 2 + 1);
    const int64_t blocks = std::min<int64_t>(grid_for(total), 148 * 32);
    for (size_t k = 0; k < doms.size(); ++k) {
      if (!solves(k)) continue;
      mdg_ctx* c = doms[k];
      PmeState* s = st[k];
      cufft_check(cufftExecD2Z(s->fwd, s->grid, s->spec), "D2Z");
      const bool energy = slot >= 0 && root(k);
      if (energy) ensure_partials(c, blocks);
      MDG_LAUNCH(c, "pme_convolve", (unsigned)blocks, kBlock, 0, k_pme_convolve, g, alpha,
                 s->bmod, s->spec, energy ? c->partials : (double*)nullptr);
      if (energy) finalize_partials(c, blocks, 1, slot, electric);
      cufft_check(cufftExecZ2D(s->inv, s->spec, s->grid), "Z2D");
    }
  }
};

void run_pme_mpole_multi(const std::vector<mdg_ctx*>& doms, PcgComm* comm, double alpha, int k1,
                         int k2, int k3, int order, double electric, bool exclude, bool ind,
                         bool forces) {
  // the combined-set pass runs on the main stream after the solve: own state
  PmeDoms P(doms, comm, ind, k1, k2, k3, order);
  const int wf = forces ? 1 : 0;
  for (size_t k = 0; k < doms.size(); ++k) {
    mdg_ctx* c = doms[k];
    P.clear(k);
    MDG_LAUNCH(c, "pme_spread_mp", grid_for(c->n_own, 128), 128, 0, k_pme_spread_mp, c->n_own,
               P.g, c->pos, c->pq4, c->mp, P.st[k]->grid, ind ? c->mu : (const double4*)nullptr);
  }
  P.sum();
  P.solve(alpha, electric, ind ? -1 : 80);
  for (size_t k = 0; k < doms.size(); ++k) {
    mdg_ctx* c = doms[k];
    const int64_t n = c->n_own;
    const double4* mu = ind ? c->mu : nullptr;
    ensure_partials(c, grid_for(n));
    MDG_LAUNCH(c, "pme_gather_mp", grid_for(n), kBlock, 0, k_pme_gather_mp, n, P.g, c->pos,
               c->pq4, c->mp, P.phi(k), electric, c->force, c->torque, c->partials, mu, wf);
    if (!ind) {
      finalize_partials(c, grid_for(n), 1, 98, 1.0);
      MDG_LAUNCH(c, "pme_self_mp", grid_for(n), kBlock, 0, k_pme_self_mp, n, c->pq4, c->mp,
                 c->partials);
      finalize_partials(c, grid_for(n), 3, 104, 1.0);  // 104 q^2, 105 mu^2, 106 Q:Q
    }
    if (exclude && c->has_mol && c->excl_start) {
      MDG_LAUNCH(c, "pme_excluded_mp", grid_for(n), kBlock, 0, k_pme_excluded_mp, n,
                 make_box(c->lx, c->ly, c->lz), alpha, electric, c->pos, c->pq4, c->mp,
                 c->excl_start, c->excl, c->force, c->torque, c->partials, mu, wf);
      if (!ind) finalize_partials(c, grid_for(n), 1, 88, 1.0);
    }
  }
}

void run_pme_mpole(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order,
                   double electric, bool exclude, const double4* ind, bool forces) {
  if (ind && ind != c->mu) throw_error(MDG_CONTRACT, "run_pme_mpole: induced set must be c->mu");
  run_pme_mpole_multi({c}, nullptr, alpha, k1, k2, k3, order, electric, exclude, ind != nullptr,
                      forces);
}

// ---- reciprocal-space electric fields for the polarization (8(f)#3) ----------
// E_i = -grad phi(r_i) from (a) the permanent multipoles (the PCG right-hand
// side) or (b) a dipole vector v (the PCG operator), plus the Ewald self field
// (4 a^3 / (3 sqrt(pi))) mu_i; the real-space kernels' Thole-damped erfc
// tensors then complete the full Ewald + Thole field. Own PME state
// (c->pme_pol): the permanent-multipole PME of the step runs on the aux
// stream at the same time.

// dipoles only: grid += sum_a v_a (K_a/L_a) dW/du_a
__global__ void k_pme_spread_dip(int64_t n, PmeGeom g, const double4* __restrict__ pos,
                                 const double4* __restrict__ v, double* __restrict__ grid,
                                 const double* __restrict__ res, int skip_converged) {
  if (skip_converged && res[27] != 0.0) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 r = pos[i];
  const double4 m = v[i];
  const double d1 = m.x * g.k1 / g.l1, d2 = m.y * g.k2 / g.l2, d3 = m.z * g.k3 / g.l3;
  int i1, i2, i3;
  double w1, w2, w3;
  frac(r.x, g.l1, g.k1, i1, w1);
  frac(r.y, g.l2, g.k2, i2, w2);
  frac(r.z, g.l3, g.k3, i3, w3);
  double t1[kMaxOrder], t2[kMaxOrder], t3[kMaxOrder], e1[kMaxOrder], e2[kMaxOrder],
      e3[kMaxOrder];
  bspline(w1, g.p, t1, e1);
  bspline(w2, g.p, t2, e2);
  bspline(w3, g.p, t3, e3);
  for (int a = 0; a < g.p; ++a) {
    const int x = (i1 - a + g.k1) % g.k1;
    for (int b = 0; b < g.p; ++b) {
      const int y = (i2 - b + g.k2) % g.k2;
      const double c0 = d1 * e1[a] * t2[b] + d2 * t1[a] * e2[b];
      const double c1 = d3 * t1[a] * t2[b];
      double* row = grid + ((size_t)x * g.k2 + y) * g.k3;
      for (int c = 0; c < g.p; ++c)
        atomicAdd(row + (i3 - c + g.k3) % g.k3, c0 * t3[c] + c1 * e3[c]);
    }
  }
}

// mode 0 (permanent): out += E + cself mu_perm (dipole of mp)
// mode 1 (add): out += E + cself v
// mode 2 (PCG): out -= E + cself v, partials p.out (p = v)
__global__ void __launch_bounds__(kBlock) k_pme_gather_field(int64_t n, PmeGeom g,
                                                            const double4* __restrict__ pos,
                                                            const double* __restrict__ phi,
                                                            const double4* __restrict__ v,
                                                            const double4* __restrict__ mp,
                                                            double cself, int mode,
                                                            double4* __restrict__ out,
                                                            double* __restrict__ partials,
                                                            const double* __restrict__ res) {
  if (mode == 2 && res[27] != 0.0) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[1] = {0.0};
  if (i < n) {
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
    const double4 m = (mode == 0) ? mp[3 * i] : v[i];
    const double ex = -gx * g.k1 / g.l1 + cself * m.x;
    const double ey = -gy * g.k2 / g.l2 + cself * m.y;
    const double ez = -gz * g.k3 / g.l3 + cself * m.z;
    double4 o = out[i];
    if (mode == 2) {
      o.x -= ex;
      o.y -= ey;
      o.z -= ez;
      acc[0] = m.x * o.x + m.y * o.y + m.z * o.z;
    } else {
      o.x += ex;
      o.y += ey;
      o.z += ez;
    }
    out[i] = o;
  }
  if (mode == 2) block_store_partials<1>(acc, partials);
}

// out_i -= erf(a r)/r-kernel field at i of the multipoles of its same-molecule
// partners (excluded from the real-space field, contained in the reciprocal one)
__global__ void k_field_excl_erf(int64_t n, Box bx, double alpha, const double4* __restrict__ pos,
                                 const double4* __restrict__ pq4, const double4* __restrict__ mp,
                                 const int32_t* __restrict__ xs, const int32_t* __restrict__ xl,
                                 double4* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 pi = pos[i];
  double ex = 0, ey = 0, ez = 0;
  for (int32_t k = xs[i]; k < xs[i + 1]; ++k) {
    const int32_t j = xl[k];
    const double4 pj = pos[j];
    double x, y, z;
    const double r2 = min_image(bx, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, x, y, z);
    const double r = sqrt(r2);
    const double inv_r = 1.0 / r, inv_r2 = inv_r * inv_r;
    double B[4];
    ewald_bn<3>(r, inv_r, inv_r2, alpha, B);
    double bare = inv_r;
    for (int q = 0; q < 4; ++q) {
      if (q > 0) bare *= (double)(2 * q - 1) * inv_r2;
      B[q] = bare - B[q];
    }
    const double qj = pq4[j].z;
    const double4 m0 = mp[3 * (size_t)j], m1 = mp[3 * (size_t)j + 1];
    const double qzz = mp[3 * (size_t)j + 2].x;
    const double qx = m0.w * x + m1.x * y + m1.y * z;
    const double qy = m1.x * x + m1.z * y + m1.w * z;
    const double qz = m1.y * x + m1.w * y + qzz * z;
    const double dr = m0.x * x + m0.y * y + m0.z * z;
    const double qr = x * qx + y * qy + z * qz;
    const double cc = B[1] * qj + B[2] * dr + B[3] * qr;
    ex += cc * x - B[1] * m0.x - 2.0 * B[2] * qx;
    ey += cc * y - B[1] * m0.y - 2.0 * B[2] * qy;
    ez += cc * z - B[1] * m0.z - 2.0 * B[2] * qz;
  }
  double4 o = out[i];
  o.x -= ex;
  o.y -= ey;
  o.z -= ez;
  out[i] = o;
}

// Reciprocal + self field added to (mode 0/1) or, in PCG form, subtracted from
// `out` with the partials of p.out (mode 2). v: the dipole vector (modes 1/2).
// The launches are capture-safe (fixed grids, no host sync).
void pme_field_multi(const std::vector<mdg_ctx*>& doms, PcgComm* comm, int mode) {
  const PolarRecip& R = doms[0]->pol_recip;
  PmeDoms P(doms, comm, true, R.k1, R.k2, R.k3, R.order);
  const double a = R.alpha;
  const double cself = 4.0 * a * a * a / (3.0 * std::sqrt(M_PI));
  auto vin = [&](mdg_ctx* c) -> const double4* {
    return mode == 0 ? nullptr : mode == 1 ? c->mu : c->cg_p;
  };
  for (size_t k = 0; k < doms.size(); ++k) {
    mdg_ctx* c = doms[k];
    const int64_t n = c->n_own;
    // (inside the PCG the partials already cover grid_for(n): no reallocation)
    if (mode == 0) ensure_partials(c, grid_for(n));
    P.clear(k);
    if (mode == 0)
      MDG_LAUNCH(c, "pme_spread_mp", grid_for(n, 128), 128, 0, k_pme_spread_mp, n, P.g, c->pos,
                 c->pq4, c->mp, P.st[k]->grid, (const double4*)nullptr);
    else
      MDG_LAUNCH(c, "pme_spread_dip", grid_for(n, 128), 128, 0, k_pme_spread_dip, n, P.g,
                 c->pos, vin(c), P.st[k]->grid, c->results, mode == 2 ? 1 : 0);
  }
  P.sum();
  P.solve(a, 1.0, -1);
  for (size_t k = 0; k < doms.size(); ++k) {
    mdg_ctx* c = doms[k];
    const int64_t n = c->n_own;
    double4* out = mode == 0 ? c->eperm : c->cg_q;
    MDG_LAUNCH(c, "pme_gather_field", grid_for(n), kBlock, 0, k_pme_gather_field, n, P.g, c->pos,
               P.phi(k), vin(c), c->mp, cself, mode, out, c->partials, c->results);
    if (mode == 0 && R.exclude && c->has_mol && c->excl_start)
      MDG_LAUNCH(c, "field_excl_erf", grid_for(n, 128), 128, 0, k_field_excl_erf, n,
                 make_box(c->lx, c->ly, c->lz), a, c->pos, c->pq4, c->mp, c->excl_start,
                 c->excl, out);
  }
}

void pme_field(mdg_ctx* c, int mode, const double4* v, double4* out) {
  const bool std_args = mode == 0 ? (v == nullptr && out == c->eperm)
                                  : (v == (mode == 1 ? c->mu : c->cg_p) && out == c->cg_q);
  if (!std_args) throw_error(MDG_CONTRACT, "pme_field: unexpected vectors");
  pme_field_multi({c}, nullptr, mode);
}
}  // namespace mdg
