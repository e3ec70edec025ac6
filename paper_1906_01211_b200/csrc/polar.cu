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
#include <cstdio>
#include <cstring>

#include <cub/cub.cuh>

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
  // CLMAP: the pair tensors go to the site clusters' U75 slots (cluster.cu)
  const uint16_t* __restrict__ cmap;  // row slot -> union position
  int32_t mstride;
  ClChunk* __restrict__ cst;  // cluster chunks: site i's tensors in cst[i / kCl][*].ten[i % kCl]
  int32_t nch, tcap;
};

// Field at i of the multipole (qj, m0.xyz = dipole, m0.w m1 qzz = Q) of j,
// R = r_i - r_j (Tinker's stored Q = Theta/3):
// E = R (rr3 q + rr5 mu.R + rr7 R.Q.R) - rr3 mu - 2 rr5 Q R
__device__ __forceinline__ void mpole_field_v(const double4& m0, const double4& m1, double qzz,
                                              double qj, double dx, double dy, double dz,
                                              double rr3, double rr5, double rr7, double& ex,
                                              double& ey, double& ez) {
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

__device__ __forceinline__ void mpole_field(const double4* __restrict__ mp, int32_t j, double qj,
                                            double dx, double dy, double dz, double rr3,
                                            double rr5, double rr7, double& ex, double& ey,
                                            double& ez) {
  const double4 m0 = ldg4(mp + 3 * (size_t)j);
  const double4 m1 = ldg4(mp + 3 * (size_t)j + 1);
  const double qzz = __ldg(&mp[3 * (size_t)j + 2].x);
  mpole_field_v(m0, m1, qzz, qj, dx, dy, dz, rr3, rr5, rr7, ex, ey, ez);
}

// TPRE: also write the pruned row (all pairs within the cutoff, exclusion
// flag in bit 31) and its T tensors; the field skips excluded pairs.
// CLMAP (with TPRE, DIRECT): the tensors of row slot h go to the site's
// cluster slot cmap[h] (cluster.cu), a zero tensor when the pair is beyond
// the cutoff, instead of beside the pruned row.
template <bool EWALD, bool MPOLE, bool EXCL, bool TPRE, bool DIRECT = false, bool CLMAP = false>
__global__ void __launch_bounds__(kBlock, MDG_PF_MINB) k_perm_field(FKArgs a) {
  static_assert(!CLMAP || (TPRE && DIRECT), "cluster slots need the direct TPRE walk");
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
    double2* trow = (TPRE && !CLMAP) ? a.trr + (size_t)i * a.pcap : nullptr;
    const uint16_t* mrow = CLMAP ? a.cmap + (size_t)i * a.mstride : nullptr;
    ClChunk* cch = CLMAP ? a.cst + (size_t)(i / kCl) * a.nch : nullptr;
    const int ct_site = (int)(i % kCl);
    int rslot = lane - 32;  // CLMAP: the row slot of this lane's chunk
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
        if (!CLMAP) trow[slot] = make_double2(rr3, rr5);
      }
      if (CLMAP) {
        const int m = mrow[rslot];
        if (m < a.tcap) cch[m >> 5].ten[ct_site][m & 31] = make_double2(rr3, rr5);
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
          if (CLMAP) {
            rslot += 32;
            if (!in) {
              const int m = mrow[rslot];
              if (m < a.tcap) cch[m >> 5].ten[ct_site][m & 31] = make_double2(0.0, 0.0);
            }
          }
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
                     double4* out, const ListView* rows = nullptr) {
  const DevList& L = c->lists[list_id];
  FKArgs k;
  k.n_i = c->n_own;
  k.pos = c->pos;
  k.polp = c->polp;
  k.pq4 = c->pq4;
  k.mp = c->mp;
  k.mol = c->mol;
  k.L = rows ? *rows : kernel_rows(c, list_id, cutoff);
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = cutoff * cutoff;
  k.alpha = alpha;
  k.thole_a = thole_a;
  k.out = out;
  k.pnbr = nullptr;
  k.trr = nullptr;
  k.pcnt = nullptr;
  k.pcap = 0;
  k.cmap = nullptr;
  k.mstride = 0;
  k.cst = nullptr;
  k.nch = 0;
  k.tcap = 0;
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
  const double dens = (double)c->n_global / vol * 4.18879020478639;
  const double expect = dens * cutoff * cutoff * cutoff;
  int32_t cap = (int32_t)std::min<double>(L.cap, 1.3 * expect + 40.0);
  cap = std::max<int32_t>(32, (cap + 31) & ~31);
  if (P.cap > cap) cap = std::min(P.cap, L.cap);
  const bool mp = c->has_mpoles, ex = exclude && c->has_mol;
  // site clusters: the unions of the rows walked (gated on the device by the
  // rows' cut generation) before the pass, which writes the tensors into
  // their cluster slots instead of beside the pruned rows
  const ListView rows = kernel_rows(c, list_id, cutoff);
  const double rb = cutoff + 0.5;  // the buffered rows' radius (kernel_rows)
  int32_t tcap = (int32_t)std::max<double>(32.0, 1.3 * dens * rb * rb * rb + 64.0);
  tcap = (tcap + 31) & ~31;
  if (P.tcap > tcap) tcap = P.tcap;
  bool force = false;
  for (int attempt = 0; attempt < 3; ++attempt) {
    const bool cl = build_clusters(c, cutoff, rows, rows.dense ? L.inner.gen : nullptr, tcap,
                                   force);
    const size_t need = (size_t)n * (size_t)cap;
    if (need > P.elems || (!cl && !P.trr)) {
      if (P.nbr) cudaFree(P.nbr);
      if (P.trr) cudaFree(P.trr);
      P.nbr = nullptr;
      P.trr = nullptr;
      MDG_CUDA_CHECK(cudaMalloc(&P.nbr, need * sizeof(int32_t)));
      // per-site tensors only for the per-site mat-vec
      if (!cl) MDG_CUDA_CHECK(cudaMalloc(&P.trr, need * sizeof(double2)));
      P.elems = need;
    }
    if (!P.cnt) MDG_CUDA_CHECK(cudaMalloc(&P.cnt, (size_t)c->n_cap * sizeof(int32_t)));
    P.cap = cap;
    FKArgs k = f_args(c, list_id, alpha, cutoff, thole_a, c->eperm, &rows);
    k.pnbr = P.nbr;
    k.trr = P.trr;
    k.pcnt = P.cnt;
    k.pcap = cap;
    if (cl) {
      k.cmap = P.cmap;
      k.mstride = P.mstride;
      k.cst = P.cst;
      k.nch = P.nch;
      k.tcap = P.tcap;
#define TPRE_CL(M, X) MDG_LAUNCH_SITES(c, "field_tpre", n, k, (k_perm_field<true, M, X, true, true, true>));
      if (mp && ex) { TPRE_CL(true, true) }
      else if (mp) { TPRE_CL(true, false) }
      else if (ex) { TPRE_CL(false, true) }
      else { TPRE_CL(false, false) }
#undef TPRE_CL
      count_stats_n(c, P.ucnt, P.ncl, 64);
    } else {
      // rows longer than cap are counted, not written; the retry below grows cap
#define TPRE_LAUNCH(M, X)                                                                     \
  if (k.L.dense) MDG_LAUNCH_SITES(c, "field_tpre", n, k, (k_perm_field<true, M, X, true, true>)); \
  else MDG_LAUNCH_SITES(c, "field_tpre", n, k, (k_perm_field<true, M, X, true, false>));
      if (mp && ex) { TPRE_LAUNCH(true, true) }
      else if (mp) { TPRE_LAUNCH(true, false) }
      else if (ex) { TPRE_LAUNCH(false, true) }
      else { TPRE_LAUNCH(false, false) }
#undef TPRE_LAUNCH
    }
    count_stats(c, P.cnt, 62);
    fetch_results(c);
    const int32_t mx = (int32_t)c->h_results[62];
    const int32_t umx = cl ? (int32_t)c->h_results[64] : 0;
    if (mx <= cap && umx <= tcap) {
      P.valid = true;
      P.sorted = rows.sorted;  // the rows walked (buffered cut or the list)
      P.src = list_id;
      P.cutoff = cutoff;
      P.directed = (int64_t)c->h_results[63];
      P.cl_valid = cl;
      static const int cl_stats = env_int("MDG_CL_STATS", 0);
      if (cl_stats && cl)
        std::fprintf(stderr, "[mdg] clusters %lld (mol order %d): U75 entries max %d mean %.1f, "
                     "tcap %d; pruned rows max %d mean %.1f\n", (long long)P.ncl,
                     (int)c->mol_sorted, umx, c->h_results[65] / (double)P.ncl, tcap, mx,
                     c->h_results[63] / (double)n);
      debug_check_rows(c, "pruned", P.nbr, P.cnt, P.cap, n, c->n, P.sorted);
      return;
    }
    if (mx > cap) cap = (mx + 31) & ~31;
    if (umx > tcap) {
      tcap = (umx + 31) & ~31;
      force = true;  // the unions' zero tensors in the new layout
    }
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
  const double* __restrict__ res;  // PCG: result slots (converged flag 27)
  // site subset (interior/halo overlap): 0 all n sites; 1 the boundary sites
  // sites[0, *nsel); 2 the interior sites sites[*nsel, n). The grid is sized
  // for n either way (warps past the subset return).
  int part;
  const int32_t* __restrict__ sites;
  const int* __restrict__ nsel;
};

// E_i = sum_j rr5 (v_j . R) R - rr3 v_j from the stored tensors; the PCG form
// writes q = p/alpha - T p and the block partial of p.q.
// SUB: the site subset of a.part (interior/halo overlap); its own
// instantiation, so the plain mat-vec keeps its code
template <bool PCG, bool SUB = false>
__global__ void __launch_bounds__(kBlock) k_tmatvec_pre(TPArgs a) {
  if (PCG && a.res[27] != 0.0) return;  // converged (speculative iteration)
  const int lane = threadIdx.x & 31;
  double acc[1] = {0.0};
  int64_t nsub = a.n;
  const int32_t* map = nullptr;
  if (SUB) {
    const int64_t nb = *a.nsel;
    nsub = a.part == 1 ? nb : a.n - nb;
    map = a.part == 1 ? a.sites : a.sites + nb;
  }
  MDG_SITE_LOOP(w, nsub, a.ipw) {
    const int64_t i = SUB ? (int64_t)map[w] : w;
    const double4 pi = a.pos[i];
    const int cnt = a.pcnt[i];
    MDG_DASSERT(cnt >= 0 && cnt <= a.pcap);
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

// ---- TMA-staged mat-vec --------------------------------------------------------
// The same product as k_tmatvec_pre, with each row's indices and pair
// tensors brought into shared memory by bulk asynchronous copies (TMA,
// cp.async.bulk + mbarrier transaction counts): while a warp computes row k
// from shared memory, the copy engine is already fetching row k + 1, so the
// row stream's HBM latency leaves the dependence chain (ncu on the LDG
// version: the largest stall is the index load feeding the gathers) and the
// only LSU global traffic left is the neighbour gathers. Two stages per
// warp; lane 0 arms the stage's barrier and issues both copies.
// dynamic shared memory of one block: barriers, then per warp two stages of
// {tensors[cap] double2, indices[cap] int32}
__host__ __device__ inline size_t tma_stage_bytes(int32_t cap) { return (size_t)cap * 20; }
__host__ __device__ inline size_t tma_warp_bytes(int32_t cap) { return (2 * tma_stage_bytes(cap) + 127) & ~(size_t)127; }
__host__ __device__ inline size_t tma_smem_bytes(int32_t cap) { return 128 + kWarps * tma_warp_bytes(cap); }

template <bool PCG>
__global__ void __launch_bounds__(kBlock) k_tmatvec_tma(TPArgs a) {
  if (PCG && a.res[27] != 0.0) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t cap = a.pcap;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + 2 * w;
  unsigned char* wb = smem + 128 + (size_t)w * tma_warp_bytes(cap);
  const size_t sb = tma_stage_bytes(cap);
  auto srr = [&](int st) { return reinterpret_cast<double2*>(wb + st * sb); };
  auto sidx = [&](int st) { return reinterpret_cast<int32_t*>(wb + st * sb + (size_t)cap * 16); };
  const int64_t first = (int64_t)blockIdx.x * a.ipw + w;
  const int64_t end = min((int64_t)a.n, ((int64_t)blockIdx.x + 1) * a.ipw);
  if (lane == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int64_t site, int st) {  // lane 0
    const int c = a.pcnt[site];
    const uint32_t bi = (uint32_t)((c * 4 + 15) & ~15), br = (uint32_t)c * 16u;
    mbar_arm(&bar[st], bi + br);
    if (c > 0) {
      bulk_load(srr(st), a.trr + (size_t)site * cap, br, &bar[st]);
      bulk_load(sidx(st), a.pnbr + (size_t)site * cap, bi, &bar[st]);
    }
  };
  if (lane == 0 && first < end) issue(first, 0);
  uint32_t phases = 0u;  // bit st: parity of stage st's next completion
  double acc[1] = {0.0};
  int k = 0;
  for (int64_t i = first; i < end; i += kWarps, ++k) {
    const int st = k & 1;
    const int64_t nxt = i + kWarps;
    if (lane == 0 && nxt < end) {
      // stage st ^ 1 was last read by the generic proxy in iteration k - 1
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(nxt, st ^ 1);
    }
    const double4 pi = a.pos[i];
    const int cnt = a.pcnt[i];
    MDG_DASSERT(cnt >= 0 && cnt <= cap);
    mbar_wait(&bar[st], (phases >> st) & 1u);
    phases ^= 1u << st;
    const int32_t* row = sidx(st);
    const double2* trow = srr(st);
    double ex = 0, ey = 0, ez = 0;
    for (int k0 = lane; k0 < cnt; k0 += 32) {
      const int32_t j = row[k0] & 0x7fffffff;
      const double2 rr = trow[k0];
      const double4 pj = ldg4(a.pos + j);
      const double4 mj = ldg4(a.in + j);
      double dx, dy, dz;
      min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
      const double dot = mj.x * dx + mj.y * dy + mj.z * dz;
      ex += rr.y * dot * dx - rr.x * mj.x;
      ey += rr.y * dot * dy - rr.x * mj.y;
      ez += rr.y * dot * dz - rr.x * mj.z;
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
    __syncwarp();
  }
  if (PCG) block_store_partials<1>(acc, a.partials);
}

// launch shape of the TMA mat-vec: (sites per block, blocks, smem bytes)
struct TmaShape {
  int64_t ipb = 0, grid = 0;
  size_t smem = 0;
};

static TmaShape tma_shape(mdg_ctx* c, int64_t n, int32_t cap) {
  TmaShape t;
  t.smem = tma_smem_bytes(cap);
  static size_t configured = 0;
  if (t.smem > configured) {
    for (const void* f : {(const void*)k_tmatvec_tma<true>, (const void*)k_tmatvec_tma<false>})
      MDG_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)t.smem));
    configured = t.smem;
  }
  int occ = 0, sms = 0, dev = 0;
  MDG_CUDA_CHECK(cudaGetDevice(&dev));
  MDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tmatvec_tma<true>, kBlock,
                                                               t.smem));
  static const int waves = env_int("MDG_TMA_WAVES", 16);
  const int64_t blocks = (int64_t)sms * std::max(1, occ) * waves;
  t.ipb = std::max<int64_t>(kWarps, (n + blocks - 1) / blocks);
  t.grid = (n + t.ipb - 1) / t.ipb;
  ensure_partials(c, t.grid);
  return t;
}

static bool use_tma(const PrunedList& P) {
  static const int on = env_int("MDG_TMA_MATVEC", 0);  // opt-in: measured slower (DESIGN 4)
  return on && tma_smem_bytes(P.cap) <= 200 * 1024;
}

// ---- PCG vector kernels ------------------------------------------------------
// result slots: 20 p.q, 21 r.z (current), 22 r.z (new), 23 sum|dmu|^2, 24 beta,
// 25 rms (D), 27 converged flag, 28 iterations. The scalar kernels form the
// LOCAL sums of a domain; a multi-domain solve sums slots 20-23 over all
// domains (PcgComm::allreduce) before the recurrences read them, so every
// domain takes identical steps. Once converged, the kernels of any further
// (speculatively queued) iteration return at once.
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
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock) {
    const double al = polp[i].x;
    const double4 E = e[i], T = t[i], m = mu[i];
    const double inva = 1.0 / al;
    const double rx = E.x - (m.x * inva - T.x), ry = E.y - (m.y * inva - T.y),
                 rz = E.z - (m.z * inva - T.z);
    r[i] = make_double4(rx, ry, rz, 0.0);
    const double4 zz = make_double4(al * rx, al * ry, al * rz, 0.0);
    z[i] = zz;
    p[i] = zz;
    acc[0] += rx * zz.x + ry * zz.y + rz * zz.z;
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

// ASPC predictor (Kolafa, J. Comput. Chem. 25, 335 (2004); the
// "Beeman/ASPC" setup of /root/reference/PAPER.md:783): the start of the
// solve extrapolated from the last converged dipoles, newest first,
// mu0 = sum_j B_j mu(t - j), B_j = (-1)^(j+1) j C(2k+4, k+2-j) / C(2k+2, k+1)
// with k = 4 (6 vectors): 22/7, -55/14, 55/21, -22/21, 5/21, -1/42. With
// fewer stored vectors the latest one is the start. The solve still runs to
// its tolerance: only the iteration count changes.
struct AspcHist {
  const double4* h[kAspcDepth];  // newest first
  int count;
};

__global__ void k_mu0_aspc(int64_t n, AspcHist hist, double4* __restrict__ mu) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (hist.count < kAspcDepth) {
    const double4 v = hist.h[0][i];
    mu[i] = make_double4(v.x, v.y, v.z, 0.0);
    return;
  }
  constexpr double B[kAspcDepth] = {22.0 / 7.0,   -55.0 / 14.0, 55.0 / 21.0,
                                    -22.0 / 21.0, 5.0 / 21.0,   -1.0 / 42.0};
  double x = 0, y = 0, z = 0;
#pragma unroll
  for (int j = 0; j < kAspcDepth; ++j) {
    const double4 v = hist.h[j][i];
    x += B[j] * v.x;
    y += B[j] * v.y;
    z += B[j] * v.z;
  }
  mu[i] = make_double4(x, y, z, 0.0);
}

// a = r.z / p.q (global sums); mu += a p; r -= a q; z = alpha r;
// partials: r.z, |a p|^2
__global__ void __launch_bounds__(kBlock) k_cg_update(int64_t n, const double2* __restrict__ polp,
                                                      const double* __restrict__ res,
                                                      const double4* __restrict__ p,
                                                      const double4* __restrict__ q,
                                                      double4* __restrict__ mu,
                                                      double4* __restrict__ r,
                                                      double4* __restrict__ z,
                                                      double* __restrict__ partials) {
  if (res[27] != 0.0) return;
  double acc[2] = {0.0, 0.0};
  // p.q == 0 only for p == 0 (r == 0: already exact); a = 0 then leaves mu
  // unchanged and the rms test stops the loop, no 0/0
  const double ak = (res[20] != 0.0) ? res[21] / res[20] : 0.0;
  // grid-stride (a grid of a few blocks per SM): few partials for the sum
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock) {
    const double al = polp[i].x;
    const double4 pp = p[i], qq = q[i], m = mu[i], rr = r[i];
    const double dx = ak * pp.x, dy = ak * pp.y, dz = ak * pp.z;
    mu[i] = make_double4(m.x + dx, m.y + dy, m.z + dz, 0.0);
    const double rx = rr.x - ak * qq.x, ry = rr.y - ak * qq.y, rz = rr.z - ak * qq.z;
    r[i] = make_double4(rx, ry, rz, 0.0);
    const double zx = al * rx, zy = al * ry, zz = al * rz;
    z[i] = make_double4(zx, zy, zz, 0.0);
    acc[0] += rx * zx + ry * zy + rz * zz;
    acc[1] += dx * dx + dy * dy + dz * dz;
  }
  block_store_partials<2>(acc, partials);
}

// p = z + beta p
__global__ void k_cg_dir(int64_t n, const double* __restrict__ res, const double4* __restrict__ z,
                         double4* __restrict__ p) {
  if (res[27] != 0.0) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double bk = res[24];
    const double4 zz = z[i], pp = p[i];
    p[i] = make_double4(zz.x + bk * pp.x, zz.y + bk * pp.y, zz.z + bk * pp.z, 0.0);
  }
}

// Fixed-order local sums of the CG partials: mode 0 r.z -> res[21] (and a
// fresh converged flag / iteration count); mode 1 p.q -> res[20]; mode 2
// r.z, sum|dmu|^2 -> res[22], res[23].
__device__ __forceinline__ void cg_finish(cudaGraphConditionalHandle h, int use_cond,
                                          double* __restrict__ res, int64_t max_iter,
                                          double n_global, double tol) {
  if (res[27] != 0.0) {
    if (use_cond) cudaGraphSetConditional(h, 0u);
    return;
  }
  const double rz_new = res[22];
  const double rms = sqrt(res[23] / n_global) * kDebye;
  res[25] = rms;
  res[24] = (res[21] != 0.0) ? rz_new / res[21] : 0.0;
  res[21] = rz_new;
  const double it = res[28] + 1.0;
  res[28] = it;
  const bool conv = rms < tol;
  res[27] = conv ? 1.0 : 0.0;
  if (use_cond) cudaGraphSetConditional(h, (!conv && it < (double)max_iter) ? 1u : 0u);
}

constexpr int kScalarThreads = 1024;
// FINISH (mode 2, one domain): then the convergence test and the loop
// condition in the same kernel (no separate one-thread launch)
template <bool FINISH = false>
__global__ void __launch_bounds__(kScalarThreads) k_cg_scalars(
    const double* __restrict__ partials, int64_t blocks, int mode, double* __restrict__ res,
    cudaGraphConditionalHandle h = {}, int use_cond = 0, int64_t max_iter = 0,
    double n_global = 0.0, double tol = 0.0) {
  if (mode != 0 && res[27] != 0.0) return;
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
      res[28] = 0.0;
    } else if (mode == 1) {
      res[20] = s[0][0];
    } else {
      res[22] = s[0][0];
      res[23] = s[1][0];
      if (FINISH) cg_finish(h, use_cond, res, max_iter, n_global, tol);
    }
  }
}

// The iteration's scalar recurrences from the (global) sums: beta, the rms
// dipole step over n_global sites, convergence, the iteration count; in the
// while graph also the loop condition.
__global__ void k_cg_finish(cudaGraphConditionalHandle h, int use_cond, double* __restrict__ res,
                            int64_t max_iter, double n_global, double tol) {
  cg_finish(h, use_cond, res, max_iter, n_global, tol);
}

__global__ void k_set_result(double* __restrict__ res, int slot, double v) { res[slot] = v; }

// One domain of a (possibly multi-domain) solve: its mat-vec arguments and
// launch shapes, fixed before any capture.
struct PcgDom {
  mdg_ctx* c;
  TPArgs k;
  CLArgs kc;
  bool cl;
  bool tma = false;
  size_t smem = 0;
  int64_t g;       // mat-vec grid
  int64_t blocks;  // vector-kernel grid
};

static void pcg_dom_setup(PcgDom& d, mdg_ctx* c) {
  const PrunedList& P = c->plist;
  const int64_t n = c->n_own;
  d.c = c;
  // vector kernels: grid-stride over a few blocks per SM, so their block
  // partials (the CG sums) stay few
  {
    static int sms = 0;
    if (sms == 0) {
      int dev = 0;
      MDG_CUDA_CHECK(cudaGetDevice(&dev));
      MDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    d.blocks = std::max<int64_t>(1, std::min<int64_t>(grid_for(n), (int64_t)sms * 8));
  }
  d.cl = P.cl_valid;
  d.tma = !d.cl && use_tma(P);
  const int64_t units = d.cl ? P.ncl : n;
  const void* kern = d.cl ? cl_matvec_kernel(true) : (const void*)k_tmatvec_pre<true>;
  int64_t ipb = sites_per_block(kern, units, c->launch_bps, c->launch_waves);
  if (d.tma) {
    const TmaShape t = tma_shape(c, n, P.cap);
    ipb = t.ipb;
    d.smem = t.smem;
  }
  d.g = (units + ipb - 1) / ipb;
  ensure_partials(c, std::max(d.g, d.blocks));
  TPArgs& k = d.k;
  k.n = n;
  k.ipw = (int)ipb;
  k.pos = c->pos;
  k.polp = c->polp;
  k.pnbr = P.nbr;
  k.pcnt = P.cnt;
  k.trr = P.trr;
  k.pcap = P.cap;
  k.b = make_box(c->lx, c->ly, c->lz);
  k.in = c->cg_p;
  k.out = c->cg_q;
  k.partials = c->partials;
  k.res = c->results;
  k.part = 0;
  k.sites = nullptr;
  k.nsel = nullptr;
  d.kc = CLArgs{};
  if (d.cl) {
    d.kc = cl_args(c, c->cg_p, c->cg_q);
    d.kc.ipw = (int)ipb;
    d.kc.partials = c->partials;
    d.kc.res = c->results;
  }
}

// boundary flag of an owned site: its pruned row holds a halo site (warp per
// site; the top bit of a row entry is a pair flag, not part of the index)
__global__ void __launch_bounds__(kBlock) k_boundary_flags(int64_t n_own, int ipw,
                                                           const int32_t* __restrict__ pnbr,
                                                           const int32_t* __restrict__ pcnt,
                                                           int32_t pcap,
                                                           uint8_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  MDG_SITE_LOOP(i, n_own, ipw) {
    const int cnt = pcnt[i];
    const int32_t* row = pnbr + (size_t)i * pcap;
    bool halo = false;
    for (int k = lane; k < cnt; k += 32) halo |= (row[k] & 0x7fffffff) >= n_own;
    const bool any = __any_sync(0xffffffffu, halo);
    if (lane == 0) flag[i] = any ? 1 : 0;
  }
}

// Interior/boundary split of a domain's owned sites for the overlapped
// exchange: c->dd_sites = the boundary sites in site order, then the
// interior ones in reverse site order (CUB's partition writes the rejected
// part backwards); *c->dd_nsel = the boundary count. Deterministic, and no
// host sync: the count stays on the device for the mat-vec launches.
static void split_sites(mdg_ctx* c) {
  const PrunedList& P = c->plist;
  const int64_t n = c->n_own;
  if (!c->dd_sites) {
    MDG_CUDA_CHECK(cudaMalloc(&c->dd_sites, (size_t)c->n_cap * sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMalloc(&c->dd_flags, (size_t)c->n_cap));
    MDG_CUDA_CHECK(cudaMalloc(&c->dd_nsel, sizeof(int)));
  }
  const int ipw = sites_per_warp(n);
  MDG_LAUNCH(c, "dd_split", warp_grid(n, ipw), kBlock, 0, k_boundary_flags, n,
             ipw * (int)kWarps, P.nbr, P.cnt, P.cap, c->dd_flags);
  cub::CountingInputIterator<int32_t> it(0);
  size_t bytes = 0;
  MDG_CUDA_CHECK(cub::DevicePartition::Flagged(nullptr, bytes, it, c->dd_flags, c->dd_sites,
                                               c->dd_nsel, (int)n, c->stream));
  if (bytes > c->dd_tmp_bytes) {
    if (c->dd_tmp) MDG_CUDA_CHECK(cudaFree(c->dd_tmp));
    MDG_CUDA_CHECK(cudaMalloc(&c->dd_tmp, bytes));
    c->dd_tmp_bytes = bytes;
  }
  MDG_CUDA_CHECK(cub::DevicePartition::Flagged(c->dd_tmp, bytes, it, c->dd_flags, c->dd_sites,
                                               c->dd_nsel, (int)n, c->stream));
}

static std::vector<mdg_ctx*> pcg_ctxs(const std::vector<PcgDom>& ds) {
  std::vector<mdg_ctx*> v;
  for (const PcgDom& d : ds) v.push_back(d.c);
  return v;
}

// The loop body, launched directly on the domains' stream (raw launches:
// also used inside stream capture, where the grids must be fixed).
// Overlapped exchange (comm->overlap(), plain mat-vec): the interior sites'
// rows run while the halo of p is refreshed on the communication stream,
// then the boundary sites'; their block partials sit side by side
// (2 g blocks, a fixed order).
static void pcg_body(std::vector<PcgDom>& ds, PcgComm* comm, cudaGraphConditionalHandle h,
                     int use_cond, int64_t max_iter, double n_global, double tol) {
  bool ov = comm && comm->overlap();
  for (const PcgDom& d : ds) ov = ov && !d.cl && !d.tma && d.c->dd_sites;
  if (ov) {
    comm->exchange_begin(MDG_VEC_P);
    for (PcgDom& d : ds) {
      TPArgs k = d.k;
      k.part = 2;
      k.sites = d.c->dd_sites;
      k.nsel = d.c->dd_nsel;
      k_tmatvec_pre<true, true><<<(unsigned)d.g, kBlock, 0, d.c->stream>>>(k);
    }
    comm->exchange_end();
  } else if (comm) {
    comm->exchange(MDG_VEC_P);
  }
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    if (ov) {
      TPArgs k = d.k;
      k.part = 1;
      k.sites = c->dd_sites;
      k.nsel = c->dd_nsel;
      k.partials = c->partials + (size_t)d.g * kRedVals;  // blocks g .. 2g - 1
      k_tmatvec_pre<true, true><<<(unsigned)d.g, kBlock, 0, c->stream>>>(k);
      c->launches++;
    } else if (d.cl) {
      cl_matvec_launch_raw(d.kc, (unsigned)d.g, c->stream);
    } else if (d.tma) {
      k_tmatvec_tma<true><<<(unsigned)d.g, kBlock, d.smem, c->stream>>>(d.k);
    } else {
      k_tmatvec_pre<true><<<(unsigned)d.g, kBlock, 0, c->stream>>>(d.k);
    }
  }
  // q -= reciprocal + self field of p (all domains' grids summed); the
  // gather rewrites the partials of p.q
  const bool recip = ds[0].c->pol_recip.on();
  if (recip) pme_field_multi(pcg_ctxs(ds), comm, 2);
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    const int64_t pb = recip ? grid_for(c->n_own) : ov ? 2 * d.g : d.g;
    k_cg_scalars<<<1, kScalarThreads, 0, c->stream>>>(c->partials, pb, 1, c->results);
  }
  if (comm) comm->allreduce(20, 1);
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    const int64_t n = c->n_own;
    k_cg_update<<<(unsigned)d.blocks, kBlock, 0, c->stream>>>(n, c->polp, c->results, c->cg_p,
                                                             c->cg_q, c->mu, c->cg_r, c->cg_z,
                                                             c->partials);
    if (comm)
      k_cg_scalars<<<1, kScalarThreads, 0, c->stream>>>(c->partials, d.blocks, 2, c->results);
    else  // one domain: the convergence test in the same kernel
      k_cg_scalars<true><<<1, kScalarThreads, 0, c->stream>>>(
          c->partials, d.blocks, 2, c->results, h, use_cond, max_iter, n_global, tol);
  }
  if (comm) comm->allreduce(22, 2);
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    // the loop condition is the first domain's (identical on all of them)
    if (comm)
      k_cg_finish<<<1, 1, 0, c->stream>>>(h, use_cond && &d == &ds[0], c->results, max_iter,
                                          n_global, tol);
    k_cg_dir<<<grid_for(c->n_own, 256), 256, 0, c->stream>>>(c->n_own, c->results, c->cg_z,
                                                             c->cg_p);
  }
  for (PcgDom& d : ds) d.c->launches += comm ? 6 : 5;
}

// Loop body as a CUDA graph with a device-side while node: the host launches
// the whole solve once. Rebuilt when a captured argument changes.
struct PcgGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<uintptr_t> key;
  ~PcgGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

static std::vector<uintptr_t> pcg_key(const std::vector<PcgDom>& ds, PcgComm* comm,
                                      int64_t max_iter, double tol, double n_global) {
  std::vector<uintptr_t> key;
  auto put = [&](const void* p, size_t bytes) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t o = 0; o < bytes; o += sizeof(uintptr_t)) {
      uintptr_t w = 0;
      std::memcpy(&w, b + o, std::min(sizeof w, bytes - o));
      key.push_back(w);
    }
  };
  for (const PcgDom& d : ds) {
    put(&d.k, sizeof d.k);
    put(&d.kc, sizeof d.kc);
    key.push_back((uintptr_t)d.cl);
    key.push_back((uintptr_t)d.g);
    key.push_back((uintptr_t)d.blocks);
    key.push_back((uintptr_t)d.c->stream);
    key.push_back((uintptr_t)d.c->n_own);
  }
  key.push_back((uintptr_t)comm);
  if (comm) key.push_back(comm->generation());
  if (comm) key.push_back((uintptr_t)comm->overlap());
  key.push_back((uintptr_t)max_iter);
  put(&tol, sizeof tol);
  put(&n_global, sizeof n_global);
  return key;
}

static void pcg_graph_launch(PcgGraph& G, std::vector<PcgDom>& ds, PcgComm* comm,
                             int64_t max_iter, double n_global, double tol) {
  cudaStream_t s = ds[0].c->stream;
  for (const PcgDom& d : ds)  // a moved partials buffer would be written after its free
    if (d.k.partials != d.c->partials || (d.cl && d.kc.partials != d.c->partials))
      throw_error(MDG_CUDA, "pcg: loop arguments hold a stale partials buffer");
  std::vector<uintptr_t> key = pcg_key(ds, comm, max_iter, tol, n_global);
  if (!G.exec || key != G.key) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    if (G.graph) cudaGraphDestroy(G.graph);
    G.exec = nullptr;
    G.graph = nullptr;
    MDG_CUDA_CHECK(cudaGraphCreate(&G.graph, 0));
    cudaGraphConditionalHandle h;
    MDG_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, G.graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    MDG_CUDA_CHECK(cudaGraphAddNode(&node, G.graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    std::vector<int64_t> launches;
    for (PcgDom& d : ds) launches.push_back(d.c->launches);
    MDG_CUDA_CHECK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeRelaxed));
    pcg_body(ds, comm, h, 1, max_iter, n_global, tol);
    cudaGraph_t captured = nullptr;
    MDG_CUDA_CHECK(cudaStreamEndCapture(s, &captured));
    MDG_CUDA_CHECK(cudaGraphInstantiate(&G.exec, G.graph, 0));
    for (size_t k = 0; k < ds.size(); ++k) ds[k].c->launches = launches[k];
    G.key = key;
  }
  MDG_CUDA_CHECK(cudaGraphLaunch(G.exec, s));
}

static std::map<const void*, PcgGraph>& pcg_graphs() {
  static std::map<const void*, PcgGraph> m;  // per first context (or group)
  return m;
}

void pcg_graph_forget(const void* owner) { pcg_graphs().erase(owner); }

// PCG over the stored T tensors of every domain's pruned rows (c->eperm =
// right-hand side), all domains' kernels on one stream (a group shares its
// stream; NCCL ranks have one domain each). comm == NULL: a single domain.
// No host round trip per iteration: the loop runs as a device-side while
// graph when the communication is capturable (single domain, in-process
// domains); otherwise (NCCL) the host queues iterations in batches ahead of
// the device, whose kernels return at once after convergence, and reads the
// converged flag a batch behind.
int64_t run_pcg_multi(std::vector<mdg_ctx*> doms, PcgComm* comm, double tol_debye,
                      int64_t max_iter, double* last_rms) {
  mdg_ctx* c0 = doms[0];
  if (c0->pol_recip.on()) {
    if (!comm && (doms.size() > 1 || c0->n_own != c0->n))
      throw_error(MDG_CONTRACT, "reciprocal-space polarization of domains needs their group");
    for (mdg_ctx* c : doms) {
      const PolarRecip &a = c->pol_recip, &b = c0->pol_recip;
      if (a.k1 != b.k1 || a.k2 != b.k2 || a.k3 != b.k3 || a.order != b.order ||
          a.alpha != b.alpha || a.exclude != b.exclude || c->lx != c0->lx || c->ly != c0->ly ||
          c->lz != c0->lz)
        throw_error(MDG_CONTRACT, "reciprocal space: the domains' grids / boxes differ");
    }
  }
  double n_global = 0;
  for (mdg_ctx* c : doms) n_global += (double)c->n_own;
  if (comm) n_global = (double)comm->n_global();
  else if (c0->n_global > 0) n_global = (double)c0->n_global;
  // mat-vec shape (MDG_PCG_BPS / MDG_PCG_WAVES): leave room on every SM for
  // the aux stream's multipole blocks
  static const int pcg_bps = env_int("MDG_PCG_BPS", 0), pcg_waves = env_int("MDG_PCG_WAVES", 0);
  std::vector<PcgDom> ds(doms.size());
  const bool ov = comm && comm->overlap();
  for (size_t k = 0; k < doms.size(); ++k) {
    mdg_ctx* c = doms[k];
    const int b = c->launch_bps, w = c->launch_waves;
    c->launch_bps = pcg_bps;
    c->launch_waves = pcg_waves;
    pcg_dom_setup(ds[k], c);
    c->launch_bps = b;
    c->launch_waves = w;
    if (ov && !ds[k].cl && !ds[k].tma) {
      split_sites(c);  // after the pruned rows of this step
      ensure_partials(c, 2 * ds[k].g);
      ds[k].k.partials = c->partials;  // (ensure_partials may have moved it)
    }
  }
  // mu0 = alpha E (or the ASPC prediction), its halo, T mu0, r0 / z0 / p0
  // and r0.z0
  const bool predict = doms.size() == 1 && !comm && c0->aspc_on && c0->aspc_count > 0;
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    if (predict) {
      AspcHist h{};
      h.count = c->aspc_count;
      for (int j = 0; j < kAspcDepth; ++j)
        h.h[j] = c->aspc_hist + (size_t)((c->aspc_head - 1 - j + 2 * kAspcDepth) % kAspcDepth) *
                                    c->n_cap;
      MDG_LAUNCH(c, "cg_mu0", grid_for(c->n_own, 256), 256, 0, k_mu0_aspc, c->n_own, h, c->mu);
    } else {
      MDG_LAUNCH(c, "cg_mu0", grid_for(c->n_own, 256), 256, 0, k_mu0, c->n_own, c->polp,
                 c->eperm, c->mu);
    }
  }
  if (comm) comm->exchange(MDG_VEC_MU);
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    if (d.cl) {
      CLArgs kc = cl_args(c, c->mu, c->cg_q);
      cl_matvec_launch(c, kc, false, "tmatvec_pre");
    } else if (d.tma) {
      TPArgs k = d.k;
      k.in = c->mu;
      MDG_LAUNCH(c, "tmatvec_pre", (unsigned)d.g, kBlock, d.smem, k_tmatvec_tma<false>, k);
    } else {
      TPArgs k = d.k;
      k.in = c->mu;
      MDG_LAUNCH_SITES(c, "tmatvec_pre", k.n, k, k_tmatvec_pre<false>);
    }
  }
  if (c0->pol_recip.on()) pme_field_multi(doms, comm, 1);  // + reciprocal + self field
  for (PcgDom& d : ds) {
    mdg_ctx* c = d.c;
    MDG_LAUNCH(c, "cg_init", (unsigned)d.blocks, kBlock, 0, k_cg_init, c->n_own, c->polp,
               c->eperm, c->cg_q, c->mu, c->cg_r, c->cg_z, c->cg_p, c->partials);
    MDG_LAUNCH(c, "cg_scalars", 1, kScalarThreads, 0, k_cg_scalars, c->partials, d.blocks, 0,
               c->results);
  }
  if (comm) comm->allreduce(21, 1);
  // the T mu0 launch above sizes its own grid (site-loop shape of the
  // non-PCG kernel) and may have grown -- moved -- the partials since
  // pcg_dom_setup: the loop kernels (and the graph key) take the current one
  for (PcgDom& d : ds) {
    d.k.partials = d.c->partials;
    if (d.cl) d.kc.partials = d.c->partials;
  }
  // (the reciprocal-space field's cuFFT calls stay out of the while graph)
  const bool graph = !c0->profile && (!comm || comm->capturable()) && !c0->pol_recip.on();
  if (graph) {
    pcg_graph_launch(pcg_graphs()[comm ? (const void*)comm : (const void*)c0], ds, comm,
                     max_iter, n_global, tol_debye);
  } else if (c0->profile) {
    // kernel-by-kernel (named, event-bracketed) host loop, one check per iteration
    for (int64_t it = 1; it <= max_iter; ++it) {
      if (comm) comm->exchange(MDG_VEC_P);
      for (PcgDom& d : ds) {
        mdg_ctx* c = d.c;
        if (d.cl) {
          CLArgs kc = d.kc;
          cl_matvec_launch(c, kc, true, "tmatvec_pcg");
        } else if (d.tma) {
          MDG_LAUNCH(c, "tmatvec_pcg", (unsigned)d.g, kBlock, d.smem, k_tmatvec_tma<true>, d.k);
          c->last_grid = d.g;
        } else {
          TPArgs k = d.k;
          MDG_LAUNCH_SITES(c, "tmatvec_pcg", k.n, k, k_tmatvec_pre<true>);
        }
      }
      if (c0->pol_recip.on()) pme_field_multi(doms, comm, 2);
      for (PcgDom& d : ds) {
        mdg_ctx* c = d.c;
        const int64_t pb = c0->pol_recip.on() ? grid_for(c->n_own) : c->last_grid;
        MDG_LAUNCH(c, "cg_scalars", 1, kScalarThreads, 0, k_cg_scalars, c->partials, pb, 1,
                   c->results);
      }
      if (comm) comm->allreduce(20, 1);
      for (PcgDom& d : ds) {
        mdg_ctx* c = d.c;
        MDG_LAUNCH(c, "cg_update", (unsigned)d.blocks, kBlock, 0, k_cg_update, c->n_own,
                   c->polp, c->results, c->cg_p, c->cg_q, c->mu, c->cg_r, c->cg_z, c->partials);
        MDG_LAUNCH(c, "cg_scalars", 1, kScalarThreads, 0, k_cg_scalars, c->partials, d.blocks,
                   2, c->results);
      }
      if (comm) comm->allreduce(22, 2);
      for (PcgDom& d : ds) {
        mdg_ctx* c = d.c;
        MDG_LAUNCH(c, "cg_finish", 1, 1, 0, k_cg_finish, cudaGraphConditionalHandle{}, 0,
                   c->results, max_iter, n_global, tol_debye);
        MDG_LAUNCH(c, "cg_dir", grid_for(c->n_own, 256), 256, 0, k_cg_dir, c->n_own, c->results,
                   c->cg_z, c->cg_p);
      }
      fetch_results(c0);
      if (c0->h_results[27] != 0.0) break;
    }
  } else {
    // speculative batches: B iterations queued per batch, the flag of batch
    // k read (mapped copy behind an event) while batch k+1 runs
    constexpr int kBatch = 4;
    constexpr int kSlot = 112;  // two host copies of (27, 28, 25) at 112.. / 116..
    cudaEvent_t ev[2];
    for (auto& e : ev) MDG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct Free {
      cudaEvent_t* e;
      ~Free() {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }
    } fr{ev};
    int64_t queued = 0;
    int batch = 0, pending = 0;
    bool done = false;
    while (!done) {
      if (queued < max_iter) {
        const int64_t m = std::min<int64_t>(kBatch, max_iter - queued);
        for (int64_t q = 0; q < m; ++q)
          pcg_body(ds, comm, cudaGraphConditionalHandle{}, 0, max_iter, n_global, tol_debye);
        queued += m;
        double* h = c0->h_results + kSlot + 4 * (batch & 1);
        for (int s : {27, 28, 25})
          MDG_CUDA_CHECK(cudaMemcpyAsync(h + (s == 27 ? 0 : s == 28 ? 1 : 2), c0->results + s,
                                         sizeof(double), cudaMemcpyDeviceToHost, c0->stream));
        MDG_CUDA_CHECK(cudaEventRecord(ev[batch & 1], c0->stream));
        ++batch;
        ++pending;
      }
      // wait for the older batch in flight (the newest when nothing more is queued)
      if (pending == 2 || queued >= max_iter) {
        const int b = (pending == 2) ? batch - 2 : batch - 1;
        MDG_CUDA_CHECK(cudaEventSynchronize(ev[b & 1]));
        --pending;
        const double* h = c0->h_results + kSlot + 4 * (b & 1);
        if (h[0] != 0.0 || (queued >= max_iter && pending == 0)) done = true;
      }
    }
    MDG_CUDA_CHECK(cudaStreamSynchronize(c0->stream));
  }
  fetch_results(c0);
  check_lists_fresh(c0);
  const int64_t it = (int64_t)c0->h_results[28];
  *last_rms = c0->h_results[25];
  if (c0->h_results[27] == 0.0)
    throw_error(MDG_CONVERGENCE, "polar_solve_pcg: no convergence after max_iter");
  if (doms.size() == 1 && !comm && c0->aspc_on) {  // keep the converged dipoles
    if (!c0->aspc_hist)
      MDG_CUDA_CHECK(cudaMalloc(&c0->aspc_hist,
                                (size_t)kAspcDepth * c0->n_cap * sizeof(double4)));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c0->aspc_hist + (size_t)c0->aspc_head * c0->n_cap, c0->mu,
                                   (size_t)c0->n_own * sizeof(double4),
                                   cudaMemcpyDeviceToDevice, c0->stream));
    c0->aspc_head = (c0->aspc_head + 1) % kAspcDepth;
    c0->aspc_count = std::min(c0->aspc_count + 1, kAspcDepth);
  }
  return it;
}

int64_t run_pcg_pre(mdg_ctx* c, double tol_debye, int64_t max_iter, double* last_rms) {
  return run_pcg_multi({c}, nullptr, tol_debye, max_iter, last_rms);
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
