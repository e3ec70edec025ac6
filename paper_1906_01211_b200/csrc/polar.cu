// polar.cu -- Thole/Ewald dipole-field mat-vec, permanent multipole field,
// and the on-device induced-dipole solvers (PCG with fused dots; Jacobi).
//
// Reference: proj/src/polar_scalar.cpp:69-198 (Thole-only T, charge-only
// field, Jacobi). With alpha > 0 the pair tensors are the real-space Ewald
// ones, rr3 = B1 - (1-l3)/r^3, rr5 = B2 - 3(1-l5)/r^5, rr7 = B3 - 15(1-l7)/r^7;
// at alpha == 0 the kernels use the reference's l3/r^3, 3 l5/r^5 forms.
//
// In the AMOEBA step the 7 A kernels share one pass over the 9 A list
// (k_field_tpre): it compacts the in-range pairs into a pruned row (exclusion
// flag in the index sign bit), stores the T pair tensors (rr3, rr5) beside
// them and accumulates the permanent field. The tensors do not change during
// the solve, so every PCG mat-vec streams 20 B per pair instead of
// recomputing erfc/exp/sqrt/div: the solve is HBM-bound.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"

// field_tpre: 6 resident blocks per SM (<= 85 registers) measured fastest
// (4.25 ms vs 4.54 unconstrained at 112 registers; 4/5/7/8 slower)
#ifndef MDG_PF_MINB
#define MDG_PF_MINB 6
#endif
#ifndef MDG_TPRE_UNROLL
#define MDG_TPRE_UNROLL 1
#endif

namespace mdg {

// ---- on-the-fly T mat-vec (reference dipole_field_matvec, Ewald generalised)
struct TKArgs {
  int64_t n_i;
  int ipw;
  const double4* __restrict__ pos;
  const double2* __restrict__ polp;
  const double4* __restrict__ pq4;
  ListView L;
  Box b;
  double c2, alpha, thole_a;
  const double4* __restrict__ in;
  double4* __restrict__ out;
  double* __restrict__ partials;  // unused (launch macro contract)
};

template <bool EWALD>
__global__ void __launch_bounds__(kBlock) k_tmatvec(TKArgs a) {
  __shared__ double4 ring_mem[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  Ring ring{ring_mem[threadIdx.x >> 5], 0, 0};
  MDG_SITE_LOOP(i, a.n_i, a.ipw) {
    const double4 pi = a.pos[i];
    const double ipdi = a.pq4[i].w;
    const int cnt = a.L.cnt[i];
    const int32_t* row = list_row(a.L, i);
    double ex = 0, ey = 0, ez = 0;
    auto body = [&](const double4& e) {
      const int32_t j = ring_j(e);
      const double dx = e.x, dy = e.y, dz = e.z;
      const double r2 = dist2(dx, dy, dz);
      const double ipdj = __ldg(&a.pq4[j].w);
      const double4 mj = ldg4(a.in + j);
      const double r = sqrt(r2);
      double l3, l5;
      thole3(r * ipdi * ipdj, a.thole_a, l3, l5);
      double rr3, rr5;
      if (EWALD) {
        const double inv_r = 1.0 / r;
        const double inv_r2 = inv_r * inv_r;
        double bn[3];
        ewald_bn<2>(r, inv_r, inv_r2, a.alpha, bn);
        const double b3 = inv_r2 * inv_r;
        rr3 = bn[1] - (1.0 - l3) * b3;
        rr5 = bn[2] - (1.0 - l5) * 3.0 * b3 * inv_r2;
      } else {
        const double r3 = r2 * r;
        rr3 = l3 / r3;
        rr5 = 3.0 * l5 / (r3 * r2);
      }
      const double dot = mj.x * dx + mj.y * dy + mj.z * dz;
      ex += rr5 * dot * dx - rr3 * mj.x;
      ey += rr5 * dot * dy - rr3 * mj.y;
      ez += rr5 * dot * dz - rr3 * mj.z;
    };
    run_row(
        row, cnt, lane, a.pos, nullptr, ring,
        [&](int32_t& raw, const double4& pj, int32_t, double& dx, double& dy, double& dz) {
          raw &= 0x7fffffff;
          return min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz) <= a.c2;
        },
        [&](const double4& e, int) { body(e); });
    ex = warp_allsum(ex);
    ey = warp_allsum(ey);
    ez = warp_allsum(ez);
    if (lane == 0) a.out[i] = make_double4(ex, ey, ez, 0.0);
  }
}

void run_tmatvec(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                 const double4* in, double4* out) {
  const DevList& L = c->lists[list_id];
  TKArgs k;
  k.n_i = c->n_own;
  k.pos = c->pos;
  k.polp = c->polp;
  k.pq4 = c->pq4;
  k.L = kernel_rows(c, list_id, cutoff);
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = cutoff * cutoff;
  k.alpha = alpha;
  k.thole_a = thole_a;
  k.in = in;
  k.out = out;
  if (alpha > 0) MDG_LAUNCH_SITES(c, "tmatvec", k.n_i, k, k_tmatvec<true>);
  else MDG_LAUNCH_SITES(c, "tmatvec", k.n_i, k, k_tmatvec<false>);
}

// ---- permanent field ----------------------------------------------------------
struct FKArgs {
  int64_t n_i;
  int ipw;
  const double4* __restrict__ pos;
  const double2* __restrict__ polp;
  const double4* __restrict__ mp;
  const int32_t* __restrict__ mol;
  ListView L;
  Box b;
  double c2, alpha, thole_a;
  double4* __restrict__ out;
  // field_tpre outputs: pruned rows, T tensors, counts
  int32_t* __restrict__ pnbr;
  double2* __restrict__ trr;
  int32_t* __restrict__ pcnt;
  int32_t pcap;
  double* __restrict__ partials;  // unused (launch macro contract)
  const double4* __restrict__ pq4;
};

// Field at i of the multipole of j, R = r_i - r_j (Tinker's stored Q = Theta/3):
// E = R (rr3 q + rr5 mu.R + rr7 R.Q.R) - rr3 mu - 2 rr5 Q R
__device__ __forceinline__ void mpole_field(const double4* __restrict__ mp, int32_t j, double qj,
                                            double dx, double dy, double dz, double rr3,
                                            double rr5, double rr7, double& ex, double& ey,
                                            double& ez) {
  const double4 m0 = ldg4(mp + 3 * (size_t)j);
  const double4 m1 = ldg4(mp + 3 * (size_t)j + 1);
  const double qzz = __ldg(&mp[3 * (size_t)j + 2].x);
  const double qx = m0.w * dx + m1.x * dy + m1.y * dz;
  const double qy = m1.x * dx + m1.z * dy + m1.w * dz;
  const double qz = m1.y * dx + m1.w * dy + qzz * dz;
  const double dr = m0.x * dx + m0.y * dy + m0.z * dz;
  const double qr = dx * qx + dy * qy + dz * qz;
  const double cc = rr3 * qj + rr5 * dr + rr7 * qr;
  const double t5 = 2.0 * rr5;
  ex += cc * dx - rr3 * m0.x - t5 * qx;
  ey += cc * dy - rr3 * m0.y - t5 * qy;
  ez += cc * dz - rr3 * m0.z - t5 * qz;
}

// TPRE: also write the pruned row (all pairs within the cutoff, exclusion
// flag in bit 31) and its T tensors; the field skips excluded pairs.
template <bool EWALD, bool MPOLE, bool EXCL, bool TPRE, bool DIRECT = false>
__global__ void __launch_bounds__(kBlock, MDG_PF_MINB) k_perm_field(FKArgs a) {
  __shared__ double4 ring_mem[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  Ring ring{ring_mem[threadIdx.x >> 5], 0, 0};
  MDG_SITE_LOOP(i, a.n_i, a.ipw) {
    const double4 pi = a.pos[i];
    const double ipdi = a.pq4[i].w;
    const int32_t mi = a.mol[i];
    const int cnt = a.L.cnt[i];
    const int32_t* row = list_row(a.L, i);
    int32_t* prow = TPRE ? a.pnbr + (size_t)i * a.pcap : nullptr;
    double2* trow = TPRE ? a.trr + (size_t)i * a.pcap : nullptr;
    double ex = 0, ey = 0, ez = 0;
    auto body = [&](const double4& e, int slot) {
      const int32_t raw = ring_j(e);
      const int32_t j = raw & 0x7fffffff;
      const double dx = e.x, dy = e.y, dz = e.z;
      const double r2 = dist2(dx, dy, dz);
      // (polarizability, pdamp, charge, 1/pdamp) of j in one 32-B load
      const double4 xj = ldg4(a.pq4 + j);
      const double4 pj = make_double4(0.0, 0.0, 0.0, xj.z);
      const double inv_r = rsqrt(r2);  // one MUFU.RSQ64H + Newton, no division
      const double r = r2 * inv_r;
      const double inv_r2 = inv_r * inv_r;
      const double b1 = inv_r2 * inv_r;
      const double u = r * ipdi * xj.w;
      if (!MPOLE && !TPRE) {
        double l3, l5;
        thole3(u, a.thole_a, l3, l5);
        double rr3;
        if (EWALD) {
          double bn[2];
          ewald_bn<1>(r, inv_r, inv_r2, a.alpha, bn);
          rr3 = bn[1] - (1.0 - l3) * b1;
        } else {
          rr3 = l3 / (r2 * r);  // proj/src/polar_scalar.cpp:143
        }
        const double cq = rr3 * pj.w;
        ex += cq * dx;
        ey += cq * dy;
        ez += cq * dz;
        return;
      }
      double l3, l5, l7;
      thole7(u, a.thole_a, l3, l5, l7);
      const double b2 = 3.0 * b1 * inv_r2, b3 = 5.0 * b2 * inv_r2;
      double rr3, rr5, rr7;
      if (EWALD) {
        double bn[4];
        ewald_bn<3>(r, inv_r, inv_r2, a.alpha, bn);
        rr3 = bn[1] - (1.0 - l3) * b1;
        rr5 = bn[2] - (1.0 - l5) * b2;
        rr7 = bn[3] - (1.0 - l7) * b3;
      } else {
        rr3 = l3 * b1;
        rr5 = l5 * b2;
        rr7 = l7 * b3;
      }
      if (TPRE && slot < a.pcap) {  // overflow -> host retries larger
        prow[slot] = raw;
        trow[slot] = make_double2(rr3, rr5);
      }
      if (EXCL && raw < 0) return;
      if (MPOLE) {
        mpole_field(a.mp, j, pj.w, dx, dy, dz, rr3, rr5, rr7, ex, ey, ez);
      } else {
        const double cq = rr3 * pj.w;
        ex += cq * dx;
        ey += cq * dy;
        ez += cq * dz;
      }
    };
    const int pn = run_row<false, DIRECT>(
        row, cnt, lane, a.pos, a.mol, ring,
        [&](int32_t& raw, const double4& pj, int32_t mj, double& dx, double& dy, double& dz) {
          const int32_t j = raw & 0x7fffffff;
          bool in = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz) <= a.c2;
          const bool same = mj == mi;
          if (!TPRE && EXCL && same) in = false;
          raw = (TPRE && same) ? (j | (int32_t)0x80000000) : j;
          return in;
        },
        body);
    ex = warp_allsum(ex);
    ey = warp_allsum(ey);
    ez = warp_allsum(ez);
    if (lane == 0) {
      a.out[i] = make_double4(ex, ey, ez, 0.0);
      if (TPRE) a.pcnt[i] = pn;
    }
  }
}

static FKArgs f_args(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                     double4* out) {
  const DevList& L = c->lists[list_id];
  FKArgs k;
  k.n_i = c->n_own;
  k.pos = c->pos;
  k.polp = c->polp;
  k.pq4 = c->pq4;
  k.mp = c->mp;
  k.mol = c->mol;
  k.L = kernel_rows(c, list_id, cutoff);
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = cutoff * cutoff;
  k.alpha = alpha;
  k.thole_a = thole_a;
  k.out = out;
  k.pnbr = nullptr;
  k.trr = nullptr;
  k.pcnt = nullptr;
  k.pcap = 0;
  return k;
}

void run_perm_field(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                    int exclude, double4* out) {
  FKArgs k = f_args(c, list_id, alpha, cutoff, thole_a, out);
  const bool ew = alpha > 0, mp = c->has_mpoles, ex = exclude && c->has_mol;
#define PF_CASE(E, M, X)                                                         \
  if (ew == E && mp == M && ex == X) {                                         \
    MDG_LAUNCH_SITES(c, "perm_field", k.n_i, k, (k_perm_field<E, M, X, false>)); \
    return;                                                                    \
  }
  PF_CASE(false, false, false)
  PF_CASE(false, false, true)
  PF_CASE(false, true, false)
  PF_CASE(false, true, true)
  PF_CASE(true, false, false)
  PF_CASE(true, false, true)
  PF_CASE(true, true, false)
  PF_CASE(true, true, true)
#undef PF_CASE
}

void run_field_tpre(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                    int exclude) {
  const DevList& L = c->lists[list_id];
  PrunedList& P = c->plist;
  const int64_t n = c->n_own;
  const double vol = c->lx * c->ly * c->lz;
  const double expect = (double)c->n_global / vol * 4.18879020478639 * cutoff * cutoff * cutoff;
  int32_t cap = (int32_t)std::min<double>(L.cap, 1.3 * expect + 40.0);
  cap = std::max<int32_t>(32, (cap + 31) & ~31);
  if (P.cap > cap) cap = std::min(P.cap, L.cap);
  P.cl_valid = false;
  const bool mp = c->has_mpoles, ex = exclude && c->has_mol;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const size_t need = (size_t)n * (size_t)cap;
    if (need > P.elems) {
      if (P.nbr) cudaFree(P.nbr);
      if (P.trr) cudaFree(P.trr);
      P.nbr = nullptr;
      P.trr = nullptr;
      MDG_CUDA_CHECK(cudaMalloc(&P.nbr, need * sizeof(int32_t)));
      MDG_CUDA_CHECK(cudaMalloc(&P.trr, need * sizeof(double2)));
      P.elems = need;
    }
    if (!P.cnt) MDG_CUDA_CHECK(cudaMalloc(&P.cnt, (size_t)c->n_cap * sizeof(int32_t)));
    P.cap = cap;
    FKArgs k = f_args(c, list_id, alpha, cutoff, thole_a, c->eperm);
    k.pnbr = P.nbr;
    k.trr = P.trr;
    k.pcnt = P.cnt;
    k.pcap = cap;
    // rows longer than cap are counted, not written; the retry below grows cap
#define TPRE_LAUNCH(M, X)                                                                     \
  if (k.L.dense) MDG_LAUNCH_SITES(c, "field_tpre", n, k, (k_perm_field<true, M, X, true, true>)); \
  else MDG_LAUNCH_SITES(c, "field_tpre", n, k, (k_perm_field<true, M, X, true, false>));
    if (mp && ex) { TPRE_LAUNCH(true, true) }
    else if (mp) { TPRE_LAUNCH(true, false) }
    else if (ex) { TPRE_LAUNCH(false, true) }
    else { TPRE_LAUNCH(false, false) }
#undef TPRE_LAUNCH
    count_stats(c, P.cnt, 62);
    fetch_results(c);
    const int32_t mx = (int32_t)c->h_results[62];
    if (mx <= cap) {
      P.valid = true;
      P.sorted = k.L.sorted;  // the rows walked (buffered cut or the list)
      P.src = list_id;
      P.cutoff = cutoff;
      P.directed = (int64_t)c->h_results[63];
      build_clusters(c, cutoff);
      return;
    }
    cap = (mx + 31) & ~31;
  }
  throw_error(MDG_CUDA, "field_tpre: capacity retry failed");
}

// ---- streaming T mat-vec over the pruned rows --------------------------------
struct TPArgs {
  int64_t n;
  int ipw;
  const double4* __restrict__ pos;
  const double2* __restrict__ polp;
  const int32_t* __restrict__ pnbr;
  const int32_t* __restrict__ pcnt;
  const double2* __restrict__ trr;
  int32_t pcap;
  Box b;
  const double4* __restrict__ in;
  double4* __restrict__ out;
  double* __restrict__ partials;
};

// E_i = sum_j rr5 (v_j . R) R - rr3 v_j from the stored tensors; the PCG form
// writes q = p/alpha - T p and the block partial of p.q.
template <bool PCG>
__global__ void __launch_bounds__(kBlock) k_tmatvec_pre(TPArgs a) {
  const int lane = threadIdx.x & 31;
  double acc[1] = {0.0};
  MDG_SITE_LOOP(i, a.n, a.ipw) {
    const double4 pi = a.pos[i];
    const int cnt = a.pcnt[i];
    const int32_t* row = a.pnbr + (size_t)i * a.pcap;
    const double2* trow = a.trr + (size_t)i * a.pcap;
    double ex = 0, ey = 0, ez = 0;
    // 4 slots per lane per round: all index/tensor loads, then all gathers,
    // then the math -- 8 independent gathers in flight per lane. Slots past
    // the row end carry rr = 0 and contribute exactly 0.
    constexpr int U = MDG_TPRE_UNROLL;
    for (int k0 = lane; k0 < cnt; k0 += 32 * U) {
      int32_t jj[U];
      double2 rr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + 32 * u;
        const bool v = k < cnt;
        // streamed once per mat-vec: evict-first so the gathered positions
        // and dipoles (64 MB) stay resident in L2
        jj[u] = v ? (__ldcs(row + k) & 0x7fffffff) : (int32_t)i;
        rr[u] = v ? __ldcs(trow + k) : make_double2(0.0, 0.0);
      }
      double4 pj[U], mj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pj[u] = ldg4(a.pos + jj[u]);
        mj[u] = ldg4(a.in + jj[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double dx, dy, dz;
        min_image(a.b, pi.x, pi.y, pi.z, pj[u].x, pj[u].y, pj[u].z, dx, dy, dz);
        const double dot = mj[u].x * dx + mj[u].y * dy + mj[u].z * dz;
        ex += rr[u].y * dot * dx - rr[u].x * mj[u].x;
        ey += rr[u].y * dot * dy - rr[u].x * mj[u].y;
        ez += rr[u].y * dot * dz - rr[u].x * mj[u].z;
      }
    }
    ex = warp_allsum(ex);
    ey = warp_allsum(ey);
    ez = warp_allsum(ez);
    if (lane == 0) {
      if (PCG) {
        const double4 p = a.in[i];
        const double inva = 1.0 / a.polp[i].x;
        const double qx = p.x * inva - ex, qy = p.y * inva - ey, qz = p.z * inva - ez;
        a.out[i] = make_double4(qx, qy, qz, 0.0);
        acc[0] += p.x * qx + p.y * qy + p.z * qz;
      } else {
        a.out[i] = make_double4(ex, ey, ez, 0.0);
      }
    }
  }
  if (PCG) block_store_partials<1>(acc, a.partials);
}

// ---- PCG vector kernels ------------------------------------------------------
// result slots: 20 p.q, 21 rz_old, 22 rz_new, 23 sum|dmu|^2, 24 beta, 25 rms (D),
// 26 a_k, 27 converged flag
constexpr double kDebye = 4.80321;

// mu0 = alpha E; r0 = E - mu0/alpha + T mu0 (t = T mu0); z = alpha r; p = z
__global__ void __launch_bounds__(kBlock) k_cg_init(int64_t n, const double2* __restrict__ polp,
                                                    const double4* __restrict__ e,
                                                    const double4* __restrict__ t,
                                                    double4* __restrict__ mu,
                                                    double4* __restrict__ r,
                                                    double4* __restrict__ z,
                                                    double4* __restrict__ p,
                                                    double* __restrict__ partials) {
  const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  double acc[1] = {0.0};
  if (i < n) {
    const double al = polp[i].x;
    const double4 E = e[i], T = t[i], m = mu[i];
    const double inva = 1.0 / al;
    const double rx = E.x - (m.x * inva - T.x), ry = E.y - (m.y * inva - T.y),
                 rz = E.z - (m.z * inva - T.z);
    r[i] = make_double4(rx, ry, rz, 0.0);
    const double4 zz = make_double4(al * rx, al * ry, al * rz, 0.0);
    z[i] = zz;
    p[i] = zz;
    acc[0] = rx * zz.x + ry * zz.y + rz * zz.z;
  }
  block_store_partials<1>(acc, partials);
}

__global__ void k_mu0(int64_t n, const double2* __restrict__ polp, const double4* __restrict__ e,
                      double4* __restrict__ mu) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double al = polp[i].x;
    const double4 E = e[i];
    mu[i] = make_double4(al * E.x, al * E.y, al * E.z, 0.0);
  }
}

// mu += a p; r -= a q; z = alpha r; partials: r.z, |a p|^2
__global__ void __launch_bounds__(kBlock) k_cg_update(int64_t n, const double2* __restrict__ polp,
                                                      const double* __restrict__ res,
                                                      const double4* __restrict__ p,
                                                      const double4* __restrict__ q,
                                                      double4* __restrict__ mu,
                                                      double4* __restrict__ r,
                                                      double4* __restrict__ z,
                                                      double* __restrict__ partials) {
  const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  double acc[2] = {0.0, 0.0};
  if (i < n) {
    const double ak = res[26];
    const double al = polp[i].x;
    const double4 pp = p[i], qq = q[i], m = mu[i], rr = r[i];
    const double dx = ak * pp.x, dy = ak * pp.y, dz = ak * pp.z;
    mu[i] = make_double4(m.x + dx, m.y + dy, m.z + dz, 0.0);
    const double rx = rr.x - ak * qq.x, ry = rr.y - ak * qq.y, rz = rr.z - ak * qq.z;
    r[i] = make_double4(rx, ry, rz, 0.0);
    const double zx = al * rx, zy = al * ry, zz = al * rz;
    z[i] = make_double4(zx, zy, zz, 0.0);
    acc[0] = rx * zx + ry * zy + rz * zz;
    acc[1] = dx * dx + dy * dy + dz * dz;
  }
  block_store_partials<2>(acc, partials);
}

// p = z + beta p
__global__ void k_cg_dir(int64_t n, const double* __restrict__ res, const double4* __restrict__ z,
                         double4* __restrict__ p) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double bk = res[24];
    const double4 zz = z[i], pp = p[i];
    p[i] = make_double4(zz.x + bk * pp.x, zz.y + bk * pp.y, zz.z + bk * pp.z, 0.0);
  }
}

// Fixed-order sums of the CG partials plus the scalar recurrences.
// mode 0: rz0 -> res[21]; mode 1: p.q -> a = rz/pq -> res[26];
// mode 2: rz_new, dsum -> beta, rms, converged.
constexpr int kScalarThreads = 1024;
__global__ void __launch_bounds__(kScalarThreads) k_cg_scalars(const double* __restrict__ partials,
                                                               int64_t blocks, int mode, int64_t n,
                                                               double tol, double* __restrict__ res) {
  // one block of 1024 threads, 4 independent loads in flight per thread: the
  // iteration's critical path waits on this sum twice (was 256 threads and
  // one dependent load chain: ~20 us per call on 2e4 partials)
  __shared__ double s[2][kScalarThreads];
  const int nv = (mode == 2) ? 2 : 1;
  for (int v = 0; v < nv; ++v) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t b = threadIdx.x;
    for (; b + 3 * kScalarThreads < blocks; b += 4 * kScalarThreads) {
      a0 += partials[b * kRedVals + v];
      a1 += partials[(b + kScalarThreads) * kRedVals + v];
      a2 += partials[(b + 2 * kScalarThreads) * kRedVals + v];
      a3 += partials[(b + 3 * kScalarThreads) * kRedVals + v];
    }
    for (; b < blocks; b += kScalarThreads) a0 += partials[b * kRedVals + v];
    s[v][threadIdx.x] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int w = kScalarThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int v = 0; v < nv; ++v) s[v][threadIdx.x] += s[v][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (mode == 0) {
      res[21] = s[0][0];
      res[27] = 0.0;
    } else if (mode == 1) {
      // p.q == 0 only for p == 0 (r == 0: already exact); a_k = 0 then
      // leaves mu unchanged and the rms test stops the loop, no 0/0
      res[20] = s[0][0];
      res[26] = (s[0][0] != 0.0) ? res[21] / s[0][0] : 0.0;
    } else {
      const double rz_new = s[0][0];
      res[22] = rz_new;
      res[23] = s[1][0];
      const double rms = sqrt(s[1][0] / (double)n) * kDebye;
      res[25] = rms;
      res[24] = (res[21] != 0.0) ? rz_new / res[21] : 0.0;
      res[21] = rz_new;
      res[27] = (rms < tol) ? 1.0 : 0.0;
    }
  }
}

// Device-side loop control of the PCG while graph: count the iteration and
// continue unless converged (res[27]) or at max_iter. res[28] = iterations.
__global__ void k_pcg_continue(cudaGraphConditionalHandle h, double* __restrict__ res,
                               int64_t max_iter) {
  const double it = res[28] + 1.0;
  res[28] = it;
  cudaGraphSetConditional(h, (res[27] == 0.0 && it < (double)max_iter) ? 1u : 0u);
}

__global__ void k_set_result(double* __restrict__ res, int slot, double v) { res[slot] = v; }

// host-side value -> device result slot (stream-ordered)
static void put_result(mdg_ctx* c, int slot, double v) {
  c->h_results[slot] = v;
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->results + slot, c->h_results + slot, sizeof(double),
                                 cudaMemcpyHostToDevice, c->stream));
}

static void dd_exchange(mdg_ctx* c, int vec_id) {
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (c->comm_exchange(c->comm_user, vec_id) != 0)
    throw_error(MDG_COMM, "halo exchange callback failed");
}

void exchange_halo(mdg_ctx* c, int vec_id) {
  if (c->comm_exchange) dd_exchange(c, vec_id);
}

static void dd_allreduce(mdg_ctx* c, double* v, int nv) {
  if (c->comm_allreduce(c->comm_user, v, nv) != 0)
    throw_error(MDG_COMM, "all-reduce callback failed");
}

// The iteration loop of run_pcg_pre as a CUDA graph: a while node whose body
// is [mat-vec + p.q, alpha, update, beta/rms, continue?, direction]; the
// k_pcg_continue kernel sets the loop condition on the device, so the host
// launches the graph once and reads back the iteration count and rms. The
// kernels and their order are those of the host-driven loop below.
static int64_t pcg_device_loop(mdg_ctx* c, TPArgs& k, int64_t n, int64_t blocks,
                               double tol_debye, int64_t max_iter, double* last_rms) {
  // the mat-vec's grid (and partials) must be fixed before capture
  const bool cl = c->plist.cl_valid;
  const int64_t units = cl ? c->plist.ncl : n;
  const void* kern = cl ? cl_matvec_kernel(true) : (const void*)k_tmatvec_pre<true>;
  const int64_t ipb = sites_per_block(kern, units, c->launch_bps, c->launch_waves);
  const int64_t g = (units + ipb - 1) / ipb;
  ensure_partials(c, std::max(g, blocks));
  k.ipw = (int)ipb;
  k.partials = c->partials;
  CLArgs kc{};
  if (cl) {
    kc = cl_args(c, k.in, k.out);
    kc.ipw = (int)ipb;
    kc.partials = c->partials;
  }
  uint64_t tol_bits;
  std::memcpy(&tol_bits, &tol_debye, sizeof tol_bits);
  std::vector<uintptr_t> key = {(uintptr_t)n, (uintptr_t)k.pnbr, (uintptr_t)k.pcnt,
                                (uintptr_t)k.trr, (uintptr_t)k.pcap, (uintptr_t)c->partials,
                                (uintptr_t)ipb, (uintptr_t)max_iter,
                                (uintptr_t)tol_bits, (uintptr_t)c->stream, (uintptr_t)cl,
                                (uintptr_t)kc.ucl, (uintptr_t)kc.ucnt, (uintptr_t)kc.ucap,
                                (uintptr_t)kc.ncl};
  {  // the box is captured by value
    uint64_t w[sizeof(Box) / sizeof(uint64_t)];
    std::memcpy(w, &k.b, sizeof w);
    for (uint64_t x : w) key.push_back((uintptr_t)x);
  }
  if (!c->pcg_exec || key != c->pcg_key) {
    if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
    if (c->pcg_graph) cudaGraphDestroy(c->pcg_graph);
    c->pcg_exec = nullptr;
    c->pcg_graph = nullptr;
    MDG_CUDA_CHECK(cudaGraphCreate(&c->pcg_graph, 0));
    cudaGraphConditionalHandle h;
    MDG_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, c->pcg_graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    MDG_CUDA_CHECK(cudaGraphAddNode(&node, c->pcg_graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const int64_t launches = c->launches;
    MDG_CUDA_CHECK(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeRelaxed));
    if (cl) cl_matvec_launch_raw(kc, (unsigned)g, c->stream);
    else k_tmatvec_pre<true><<<(unsigned)g, kBlock, 0, c->stream>>>(k);
    k_cg_scalars<<<1, kScalarThreads, 0, c->stream>>>(c->partials, g, 1, n, tol_debye, c->results);
    k_cg_update<<<(unsigned)blocks, kBlock, 0, c->stream>>>(n, c->polp, c->results, c->cg_p,
                                                           c->cg_q, c->mu, c->cg_r, c->cg_z,
                                                           c->partials);
    k_cg_scalars<<<1, kScalarThreads, 0, c->stream>>>(c->partials, blocks, 2, n, tol_debye, c->results);
    k_pcg_continue<<<1, 1, 0, c->stream>>>(h, c->results, max_iter);
    k_cg_dir<<<grid_for(n, 256), 256, 0, c->stream>>>(n, c->results, c->cg_z, c->cg_p);
    cudaGraph_t captured = nullptr;
    MDG_CUDA_CHECK(cudaStreamEndCapture(c->stream, &captured));
    MDG_CUDA_CHECK(cudaGraphInstantiate(&c->pcg_exec, c->pcg_graph, 0));
    c->launches = launches;
    c->pcg_key = key;
  }
  MDG_LAUNCH(c, "set_result", 1, 1, 0, k_set_result, c->results, 28, 0.0);
  MDG_CUDA_CHECK(cudaGraphLaunch(c->pcg_exec, c->stream));
  fetch_results(c);
  const int64_t it = (int64_t)c->h_results[28];
  c->launches += 6 * it;  // the body's kernels, executed on the device
  *last_rms = c->h_results[25];
  if (c->h_results[27] == 0.0)
    throw_error(MDG_CONVERGENCE, "polar_solve_pcg: no convergence after max_iter");
  return it;
}

// One PCG mat-vec over the stored tensors: the cluster kernel when the
// cluster unions are built, else the per-site stream.
static int64_t matvec_pre(mdg_ctx* c, TPArgs& k, bool pcg, const char* name) {
  if (c->plist.cl_valid) {
    CLArgs kc = cl_args(c, k.in, k.out);
    cl_matvec_launch(c, kc, pcg, name);
  } else if (pcg) {
    MDG_LAUNCH_SITES(c, name, k.n, k, k_tmatvec_pre<true>);
  } else {
    MDG_LAUNCH_SITES(c, name, k.n, k, k_tmatvec_pre<false>);
  }
  return c->last_grid;
}

// PCG over the stored T tensors. Single domain: every scalar recurrence stays
// on the device (k_cg_scalars) and the host reads one flag per iteration.
// Multi-domain (comm hooks set): the halo of mu / p is exchanged before each
// mat-vec, and the local partial sums are all-reduced on the host before the
// scalars are formed, so every rank takes identical steps.
int64_t run_pcg_pre(mdg_ctx* c, double tol_debye, int64_t max_iter, double* last_rms) {
  const int64_t n = c->n_own;
  const bool dd = c->comm_allreduce != nullptr;
  const double n_glob = (double)(c->n_global > 0 ? c->n_global : n);
  const int64_t blocks = grid_for(n);
  PrunedList& P = c->plist;
  // mat-vec shape (MDG_PCG_BPS / MDG_PCG_WAVES): leave room on every SM for
  // the aux stream's multipole blocks
  struct Shape {
    mdg_ctx* c;
    int b, w;
    ~Shape() { c->launch_bps = b; c->launch_waves = w; }
  } shape{c, c->launch_bps, c->launch_waves};
  static const int pcg_bps = env_int("MDG_PCG_BPS", 0), pcg_waves = env_int("MDG_PCG_WAVES", 0);
  c->launch_bps = pcg_bps;
  c->launch_waves = pcg_waves;
  TPArgs k;
  k.n = n;
  ensure_partials(c, blocks);
  k.pos = c->pos;
  k.polp = c->polp;
  k.pnbr = P.nbr;
  k.pcnt = P.cnt;
  k.trr = P.trr;
  k.pcap = P.cap;
  k.b = make_box(c->lx, c->ly, c->lz);
  k.partials = c->partials;
  MDG_LAUNCH(c, "cg_mu0", grid_for(n, 256), 256, 0, k_mu0, n, c->polp, c->eperm, c->mu);
  if (dd) dd_exchange(c, MDG_VEC_MU);
  k.in = c->mu;
  k.out = c->cg_q;
  matvec_pre(c, k, false, "tmatvec_pre");
  MDG_LAUNCH(c, "cg_init", (unsigned)blocks, kBlock, 0, k_cg_init, n, c->polp, c->eperm,
             c->cg_q, c->mu, c->cg_r, c->cg_z, c->cg_p, c->partials);
  MDG_LAUNCH(c, "cg_scalars", 1, kScalarThreads, 0, k_cg_scalars, c->partials, blocks, 0, n, tol_debye,
             c->results);
  double rz = 0.0;  // global r.z (multi-domain path)
  if (dd) {
    fetch_results(c);
    rz = c->h_results[21];
    dd_allreduce(c, &rz, 1);
    put_result(c, 21, rz);
  }
  k.in = c->cg_p;
  k.out = c->cg_q;
  if (!dd && !c->profile) return pcg_device_loop(c, k, n, blocks, tol_debye, max_iter, last_rms);
  k.in = c->cg_p;
  k.out = c->cg_q;
  for (int64_t it = 1; it <= max_iter; ++it) {
    if (dd) dd_exchange(c, MDG_VEC_P);
    matvec_pre(c, k, true, "tmatvec_pcg");
    MDG_LAUNCH(c, "cg_scalars", 1, kScalarThreads, 0, k_cg_scalars, c->partials, c->last_grid, 1, n,
               tol_debye, c->results);
    if (dd) {
      fetch_results(c);
      double pq = c->h_results[20];
      dd_allreduce(c, &pq, 1);
      put_result(c, 26, pq != 0.0 ? rz / pq : 0.0);  // a_k from global sums
    }
    MDG_LAUNCH(c, "cg_update", (unsigned)blocks, kBlock, 0, k_cg_update, n, c->polp, c->results,
               c->cg_p, c->cg_q, c->mu, c->cg_r, c->cg_z, c->partials);
    MDG_LAUNCH(c, "cg_scalars", 1, kScalarThreads, 0, k_cg_scalars, c->partials, blocks, 2, n, tol_debye,
               c->results);
    fetch_results(c);
    if (dd) {
      double v[2] = {c->h_results[22], c->h_results[23]};  // local rz_new, sum |dmu|^2
      dd_allreduce(c, v, 2);
      const double rms = std::sqrt(v[1] / n_glob) * kDebye;
      put_result(c, 24, rz != 0.0 ? v[0] / rz : 0.0);  // beta
      rz = v[0];
      put_result(c, 21, rz);
      *last_rms = rms;
      if (rms < tol_debye) return it;
    } else {
      *last_rms = c->h_results[25];
      if (c->h_results[27] != 0.0) return it;
    }
    MDG_LAUNCH(c, "cg_dir", grid_for(n, 256), 256, 0, k_cg_dir, n, c->results, c->cg_z, c->cg_p);
  }
  throw_error(MDG_CONVERGENCE, "polar_solve_pcg: no convergence after max_iter");
}

// ---- Jacobi (reference semantics) ------------------------------------------------
// mu_new = alpha (E + T mu); resid = max |mu_new - mu| (block max -> partials)
__global__ void __launch_bounds__(kBlock) k_jacobi_update(int64_t n, const double2* __restrict__ polp,
                                                          const double4* __restrict__ e,
                                                          const double4* __restrict__ t,
                                                          double4* __restrict__ mu,
                                                          double* __restrict__ partials) {
  const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  double m = 0.0;
  if (i < n) {
    const double al = polp[i].x;
    const double4 E = e[i], T = t[i], old = mu[i];
    const double nx = al * (E.x + T.x), ny = al * (E.y + T.y), nz = al * (E.z + T.z);
    m = fmax(fabs(nx - old.x), fmax(fabs(ny - old.y), fabs(nz - old.z)));
    mu[i] = make_double4(nx, ny, nz, 0.0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  __shared__ double red[kBlock / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) s = fmax(s, red[w]);
    partials[(size_t)blockIdx.x * kRedVals] = s;
  }
}

__global__ void k_max_partials(const double* __restrict__ partials, int64_t blocks,
                               double* __restrict__ res, int slot) {
  __shared__ double s[256];
  double m = 0.0;
  for (int64_t b = threadIdx.x; b < blocks; b += 256) m = fmax(m, partials[b * kRedVals]);
  s[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) res[slot] = s[0];
}

int64_t run_jacobi(mdg_ctx* c, int list_id, double cutoff, double thole_a, double tol,
                   int64_t max_iter, double* last_resid) {
  const int64_t n = c->n_own;
  const int64_t blocks = grid_for(n);
  ensure_partials(c, blocks);
  zero_vec(c, c->mu);
  for (int64_t it = 1; it <= max_iter; ++it) {
    run_tmatvec(c, list_id, 0.0, cutoff, thole_a, c->mu, c->cg_q);
    MDG_LAUNCH(c, "jacobi_update", (unsigned)blocks, kBlock, 0, k_jacobi_update, n, c->polp,
               c->eperm, c->cg_q, c->mu, c->partials);
    MDG_LAUNCH(c, "max_partials", 1, 256, 0, k_max_partials, c->partials, blocks, c->results, 30);
    fetch_results(c);
    *last_resid = c->h_results[30];
    if (*last_resid <= tol) return it;
  }
  throw_error(MDG_CONVERGENCE, "jacobi_polarization_solve: no convergence after max_iter");
}

}  // namespace mdg
