// nonpolar.cu -- Lennard-Jones, real-space Ewald charge and Halgren 14-7.
//
// Warp per i site over its (both-direction) row (common.cuh): the prologue
// (minimum image, cutoff, exclusion) runs on every list slot, the in-range
// pairs are ballot-compacted so the pair body runs on full warps, the i-side
// force is a warp reduction. Default (HALF): an owned-owned pair is evaluated
// once, in the row of its lower sorted index, and the partner's force is
// added with an FP64 atomic (Newton's third law, as the reference's half
// lists). Deterministic mode (!HALF): every row is summed in full, no
// atomics, each pair counted twice and the energies/virials halved in the
// fixed-order finalize.
// Pair arithmetic follows the reference: proj/include/mdvec/kernels.hpp:42-64
// (LJ, Ewald) and proj/src/polar_vec.cpp:74-116 (Halgren one-division form).
#include "common.cuh"

namespace mdg {

struct NonpolarKArgs {
  int64_t n_i;
  int ipw;
  const double4* __restrict__ pos;
  const double4* __restrict__ vdwp;
  const double4* __restrict__ vtab;  // vdW type table, or NULL: per-site vdwp of j
  const double4* __restrict__ pq4;  // charges (z)
  const double4* __restrict__ ptab;  // site-type copy of pq4, or NULL: per-site pq4 of j
  const int32_t* __restrict__ mol;
  ListView L;
  Box b;
  double c2, alpha, electric;
  double4* __restrict__ force;
  double* __restrict__ partials;
};

// partial slots: 0 E_lj, 1 E_coul, 2..7 virial (xx xy xz yy yz zz)
template <bool LJ, bool COUL, bool SHIFT, bool EXCL, bool HALF, bool DIRECT>
__global__ void __launch_bounds__(kBlock) k_nonpolar(NonpolarKArgs a) {
  __shared__ double4 ring_mem[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  Ring ring{ring_mem[threadIdx.x >> 5], 0, 0};
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double two_over_sqrt_pi = 1.1283791670955126;
  MDG_SITE_LOOP(i, a.n_i, a.ipw) {
    const double4 pi = a.pos[i];
    double4 vi = make_double4(0, 0, 0, 0);
    if (LJ) vi = a.vdwp[i];
    const double qi = COUL ? a.pq4[i].z : 0.0;
    const int cnt = a.L.cnt[i];
    const int32_t* row = list_row(a.L, i);
    double fx = 0, fy = 0, fz = 0;
    auto body = [&](const double4& e) {
      const int32_t j = ring_j(e);
      const double dx = e.x, dy = e.y, dz = e.z;
      const double r2 = dist2(dx, dy, dz);
      double fs = 0.0;
      // pair weight: 1/2 for a halo partner (the other domain has the mirror)
      const double w = (HALF && j >= a.n_i) ? 0.5 : 1.0;
      if (LJ) {
        const double4 vj = a.vtab ? ldg4(a.vtab + ring_type(e)) : ldg4(a.vdwp + j);
        const double sij = 0.5 * (vi.x + vj.x);
        const double eij = vi.y * vj.y;
        const double inv_r2 = 1.0 / r2;
        const double s2 = sij * sij * inv_r2;
        const double s6 = s2 * s2 * s2;
        const double s12 = s6 * s6;
        double u = 4.0 * eij * (s12 - s6);
        if (SHIFT) {
          const double sc2 = sij * sij / a.c2;
          const double sc6 = sc2 * sc2 * sc2;
          u -= 4.0 * eij * (sc6 * sc6 - sc6);
        }
        acc[0] += w * u;
        fs += 24.0 * eij * (2.0 * s12 - s6) * inv_r2;
      }
      if (COUL) {
        const double inv_r = rsqrt(r2);  // one MUFU.RSQ64H + Newton, no division
        const double r = r2 * inv_r;
        const double qq = a.electric * qi * __ldg(&(a.ptab ? a.ptab + ring_type(e) : a.pq4 + j)->z);
        const double ar = a.alpha * r;
        const double ex2 = exp(-ar * ar);
        const double ee = erfc_from_exp(ar, ex2) * inv_r;
        const double g = a.alpha * two_over_sqrt_pi * ex2;
        acc[1] += w * (qq * ee);
        fs += qq * (ee + g) * inv_r * inv_r;
      }
      const double px = fs * dx, py = fs * dy, pz = fs * dz;
      fx += px;
      fy += py;
      fz += pz;
      if (HALF && j < a.n_i) {
        atomicAdd(&a.force[j].x, -px);
        atomicAdd(&a.force[j].y, -py);
        atomicAdd(&a.force[j].z, -pz);
      }
      acc[2] += w * (dx * px);
      acc[3] += w * (dx * py);
      acc[4] += w * (dx * pz);
      acc[5] += w * (dy * py);
      acc[6] += w * (dy * pz);
      acc[7] += w * (dz * pz);
    };
    // half rows: a sorted row's pairs with j > i are its suffix
    const int start = (HALF && a.L.sorted) ? row_suffix(row, cnt, i, lane) : 0;
    run_row<true, DIRECT>(
        row + start, cnt - start, lane, a.pos, nullptr, ring,
        [&](int32_t j, const double4& pj, int32_t, double& dx, double& dy, double& dz) {
          const double r2 = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
          // w = exclusion group
          return (r2 <= a.c2) && !(EXCL && same_group(pj, pi)) && !(HALF && j < i);
        },
        [&](const double4& e, int) { body(e); });
    fx = warp_allsum(fx);
    fy = warp_allsum(fy);
    fz = warp_allsum(fz);
    if (lane == 0) {
      if (HALF) {
        atomicAdd(&a.force[i].x, fx);
        atomicAdd(&a.force[i].y, fy);
        atomicAdd(&a.force[i].z, fz);
      } else {
        a.force[i] = make_double4(fx, fy, fz, 0.0);
      }
    }
  }
  block_store_partials<8>(acc, a.partials);
}

template <bool LJ, bool COUL>
static void launch_np(mdg_ctx* c, const NonpolarKArgs& k, bool shift, bool excl, bool half,
                      const char* name) {
  NonpolarKArgs kk = k;
#define NP_CASE(S, E)                                                              \
  if (shift == S && excl == E) {                                                 \
    if (kk.L.dense) {                                                            \
      if (half) MDG_LAUNCH_SITES(c, name, kk.n_i, kk, (k_nonpolar<LJ, COUL, S, E, true, true>)); \
      else MDG_LAUNCH_SITES(c, name, kk.n_i, kk, (k_nonpolar<LJ, COUL, S, E, false, true>));     \
    } else {                                                                     \
      if (half) MDG_LAUNCH_SITES(c, name, kk.n_i, kk, (k_nonpolar<LJ, COUL, S, E, true, false>)); \
      else MDG_LAUNCH_SITES(c, name, kk.n_i, kk, (k_nonpolar<LJ, COUL, S, E, false, false>));    \
    }                                                                            \
    return;                                                                      \
  }
  NP_CASE(false, false)
  NP_CASE(false, true)
  NP_CASE(true, false)
  NP_CASE(true, true)
#undef NP_CASE
}

void run_nonpolar(mdg_ctx* c, int list_id, const NonpolarArgs& a) {
  const DevList& L = c->lists[list_id];
  NonpolarKArgs k;
  k.n_i = c->n_own;
  k.pos = (L.sites == MDG_SITES_VDW) ? c->vsite : c->pos;
  k.vdwp = c->vdwp;
  k.vtab = c->n_vtypes ? c->vtab : nullptr;
  k.pq4 = c->pq4;
  k.ptab = c->n_vtypes ? c->ptab : nullptr;
  k.mol = c->mol;
  k.L = kernel_rows(c, list_id, a.cutoff);
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = a.cutoff * a.cutoff;
  k.alpha = a.alpha;
  k.electric = a.electric;
  k.force = (L.sites == MDG_SITES_VDW) ? c->force2 : c->force;
  if (L.sites == MDG_SITES_VDW && a.do_coul)
    throw_error(MDG_CONTRACT, "coulomb terms need a list over atomic sites");
  const bool shift = a.shift != 0, excl = a.exclude != 0 && c->has_mol;
  const bool half = !c->deterministic;
  if (half) MDG_CUDA_CHECK(cudaMemsetAsync(k.force, 0, (size_t)k.n_i * sizeof(double4), c->stream));
  if (a.do_lj && a.do_coul) launch_np<true, true>(c, k, shift, excl, half, "lj_ewald");
  else if (a.do_lj) launch_np<true, false>(c, k, shift, excl, half, "lj");
  else launch_np<false, true>(c, k, shift, excl, half, "ewald_real");
  finalize_partials(c, c->last_grid, 8, 0, half ? 1.0 : 0.5);
}

// ---- Halgren buffered 14-7 -------------------------------------------------
struct HalgrenKArgs {
  int64_t n_i;
  int ipw;
  const double4* __restrict__ site;
  const double4* __restrict__ vdwp;
  const double4* __restrict__ vtab;  // vdW type table, or NULL: per-site vdwp of j
  const int32_t* __restrict__ mol;
  ListView L;
  Box b;
  double c2, delta, gamma;
  double4* __restrict__ force;
  double* __restrict__ partials;
};

// One Halgren buffered-14-7 pair, proj/src/polar_vec.cpp:78-107 op for op
// (all reciprocals from one division): the energy u and the force factor fs
// (the force on i is fs R, R = r_i - r_j).
__device__ __forceinline__ void halgren_pair(double r2, const double4& vi, const double4& vj,
                                         double delta, double gamma, double& u,
                                         double& fs) {
  const double r = sqrt(r2);
  const double r0 = 0.5 * (vi.z + vj.z);
  const double eij = vi.w * vj.w;
  const double r0_2 = r0 * r0;
  const double r0_3 = r0_2 * r0;
  const double r0_6 = r0_3 * r0_3;
  const double r0_7 = r0_6 * r0;
  const double r3 = r2 * r;
  const double r6 = r3 * r3;
  const double r7 = r6 * r;
  const double e1 = r + delta * r0;
  const double e2 = r7 + gamma * r0_7;
  const double r0r = r0 * r;
  const double q = 1.0 / (e1 * e2 * r0r);
  const double inv_e1 = q * e2 * r0r;
  const double inv_e2 = q * e1 * r0r;
  const double inv_r0r = q * e1 * e2;
  const double t1 = (1.0 + delta) * r0 * inv_e1;
  const double t2 = t1 * t1;
  const double t4 = t2 * t2;
  const double t7 = t4 * t2 * t1;
  const double g1 = (1.0 + gamma) * r0_7 * inv_e2;
  const double bb = g1 - 2.0;
  u = eij * t7 * bb;
  const double dudrho = -7.0 * eij * t7 * (bb * r0 * inv_e1 + r6 * r0 * g1 * inv_e2);
  fs = -dudrho * inv_r0r;
}

// HALF: each owned-owned pair once (in the row of its lower sorted index)
// with the partner's force added atomically; pairs with a halo partner stay
// in the owned row only (their mirror is the other domain's). Energy and
// virial are weighted 1 (owned pair) or 1/2 (halo pair), finalize scale 1.
// !HALF: full rows, each pair in both rows at weight 1/2 (finalize scale).
template <bool EXCL, bool HALF, bool DIRECT>
__global__ void __launch_bounds__(kBlock, MDG_HALGREN_MINB) k_halgren(HalgrenKArgs a) {
  __shared__ double4 ring_mem[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  Ring ring{ring_mem[threadIdx.x >> 5], 0, 0};
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double delta = a.delta, gamma = a.gamma;
  MDG_SITE_LOOP(i, a.n_i, a.ipw) {
    const double4 pi = a.site[i];
    const double4 vi = a.vdwp[i];
    const int cnt = a.L.cnt[i];
    const int32_t* row = list_row(a.L, i);
    double fx = 0, fy = 0, fz = 0;
    auto body = [&](const double4& e) {
      const int32_t j = ring_j(e);
      const double dx = e.x, dy = e.y, dz = e.z;
      const double r2 = dist2(dx, dy, dz);
      // j's parameters: the type table (one line shared by the warp) or j's record
      const double4 vj = a.vtab ? ldg4(a.vtab + ring_type(e)) : ldg4(a.vdwp + j);
      double u, fs;
      halgren_pair(r2, vi, vj, delta, gamma, u, fs);
      const double px = fs * dx, py = fs * dy, pz = fs * dz;
      fx += px;
      fy += py;
      fz += pz;
      double w = 1.0;
      if (HALF) {
        if (j < a.n_i) {
          atomicAdd(&a.force[j].x, -px);
          atomicAdd(&a.force[j].y, -py);
          atomicAdd(&a.force[j].z, -pz);
        } else {
          w = 0.5;
        }
      }
      acc[0] += w * u;
      acc[2] += w * (dx * px);
      acc[3] += w * (dx * py);
      acc[4] += w * (dx * pz);
      acc[5] += w * (dy * py);
      acc[6] += w * (dy * pz);
      acc[7] += w * (dz * pz);
    };
    // half rows: a sorted row's pairs with j > i are its suffix
    const int start = (HALF && a.L.sorted) ? row_suffix(row, cnt, i, lane) : 0;
    run_row<true, DIRECT>(
        row + start, cnt - start, lane, a.site, nullptr, ring,
        [&](int32_t j, const double4& pj, int32_t, double& dx, double& dy, double& dz) {
          const double r2 = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
          // w = exclusion group
          return (r2 <= a.c2) && !(EXCL && same_group(pj, pi)) && !(HALF && j < i);
        },
        [&](const double4& e, int) { body(e); });
    fx = warp_allsum(fx);
    fy = warp_allsum(fy);
    fz = warp_allsum(fz);
    if (lane == 0) {
      if (HALF) {
        atomicAdd(&a.force[i].x, fx);
        atomicAdd(&a.force[i].y, fy);
        atomicAdd(&a.force[i].z, fz);
      } else {
        a.force[i] = make_double4(fx, fy, fz, 0.0);
      }
    }
  }
  block_store_partials<8>(acc, a.partials);
}

// Halgren on site clusters (cluster.cu build_row_unions): warp per cluster
// of kCl consecutive sites (a water molecule in the molecule-keyed order),
// lane per entry j of the union of the sites' buffered rows past the
// cluster's first site (cluster.cu k_row_union), so each pair once, in the
// cluster of its lower index (the per-site half rows' rule: j > i). j's record is
// gathered and its partner force added with FP64 atomics once for the kCl
// sites (2.15 pairs per entry on config 4, against one per pair in the
// per-site rows); the sites' forces are summed once per cluster. Every pair
// within the cutoff of site t is in t's own row, so the pairs (and each
// pair's arithmetic) are those of k_halgren<HALF>.
struct HalgrenClArgs {
  int64_t n_i;  // owned sites
  int64_t ncl;
  int ipw;
  const double4* __restrict__ site;
  const double4* __restrict__ vdwp;
  const double4* __restrict__ vtab;
  const int32_t* __restrict__ uidx;
  const int32_t* __restrict__ ucnt;
  int32_t ucap;
  Box b;
  double c2, delta, gamma;
  double4* __restrict__ force;
  double* __restrict__ partials;
};

#ifndef MDG_HALGREN_CL_MINB
#define MDG_HALGREN_CL_MINB 4
#endif
template <bool EXCL>
__global__ void __launch_bounds__(kBlock, MDG_HALGREN_CL_MINB) k_halgren_cl(HalgrenClArgs a) {
  __shared__ double4 sp_mem[kWarps][kCl], sv_mem[kWarps][kCl];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double4* sp = sp_mem[w];
  double4* sv = sv_mem[w];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double delta = a.delta, gamma = a.gamma;
  MDG_SITE_LOOP(cl, a.ncl, a.ipw) {
    const int64_t i0 = cl * kCl;
    const int nv = (int)min((int64_t)kCl, a.n_i - i0);
    __syncwarp();
    if (lane < nv) {
      sp[lane] = a.site[i0 + lane];
      sv[lane] = a.vdwp[i0 + lane];
    }
    __syncwarp();
    const int ucount = a.ucnt[cl];
    const int32_t* urow = a.uidx + (size_t)cl * a.ucap;
    const int start = 0;  // the half union: every entry is past the cluster's first site
    double fx[kCl], fy[kCl], fz[kCl];
#pragma unroll
    for (int t = 0; t < kCl; ++t) fx[t] = fy[t] = fz[t] = 0.0;
    // index two chunks ahead, j's record one chunk ahead (as run_row)
    int32_t ja = (start + lane < ucount) ? __ldg(urow + start + lane) : (int32_t)i0;
    double4 pa = ldg4(a.site + ja);
    int32_t jb = (start + 32 + lane < ucount) ? __ldg(urow + start + 32 + lane) : (int32_t)i0;
    for (int base = start; base < ucount; base += 32) {
      double4 pb = make_double4(0.0, 0.0, 0.0, 0.0);
      int32_t jc = (int32_t)i0;
      if (base + 32 < ucount) pb = ldg4(a.site + jb);
      if (base + 64 + lane < ucount) jc = __ldg(urow + base + 64 + lane);
      const bool vs = base + lane < ucount;
      const int32_t j = ja;
      const double4 pj = pa;
      const double4 vj = a.vtab ? ldg4(a.vtab + __double2hiint(pj.w)) : ldg4(a.vdwp + j);
      const bool owned_j = j < a.n_i;
      const double wj = owned_j ? 1.0 : 0.5;
      double gx = 0.0, gy = 0.0, gz = 0.0;  // the partner's force
      bool any = false;
#pragma unroll
      for (int t = 0; t < kCl; ++t) {
        if (t < nv) {
          const double4 pi = sp[t];
          double dx, dy, dz;
          const double r2 = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
          const bool in = vs && j > (int32_t)(i0 + t) && (r2 <= a.c2) &&
                          !(EXCL && same_group(pj, pi));
          if (in) {
            double u, fs;
            halgren_pair(r2, sv[t], vj, delta, gamma, u, fs);
            const double px = fs * dx, py = fs * dy, pz = fs * dz;
            fx[t] += px;
            fy[t] += py;
            fz[t] += pz;
            gx -= px;
            gy -= py;
            gz -= pz;
            any = true;
            acc[0] += wj * u;
            acc[2] += wj * (dx * px);
            acc[3] += wj * (dx * py);
            acc[4] += wj * (dx * pz);
            acc[5] += wj * (dy * py);
            acc[6] += wj * (dy * pz);
            acc[7] += wj * (dz * pz);
          }
        }
      }
      if (any && owned_j) {
        atomicAdd(&a.force[j].x, gx);
        atomicAdd(&a.force[j].y, gy);
        atomicAdd(&a.force[j].z, gz);
      }
      ja = jb;
      pa = pb;
      jb = jc;
    }
#pragma unroll
    for (int t = 0; t < kCl; ++t) {
      if (t < nv) {
        const double sx = warp_allsum(fx[t]), sy = warp_allsum(fy[t]), sz = warp_allsum(fz[t]);
        if (lane == 0) {
          atomicAdd(&a.force[i0 + t].x, sx);
          atomicAdd(&a.force[i0 + t].y, sy);
          atomicAdd(&a.force[i0 + t].z, sz);
        }
      }
    }
  }
  block_store_partials<8>(acc, a.partials);
}

// F_atom[i] = f_i F_site[i] + sum over children c of (1 - f_c) F_site[c]
// (children CSR built on the host from hred_parent; sorted indices).
__global__ void k_chain_rule(int64_t n, const double4* __restrict__ fsite,
                             const int32_t* __restrict__ par, const double* __restrict__ fac,
                             const int32_t* __restrict__ child_start,
                             const int32_t* __restrict__ child, double4* __restrict__ fatom) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 fi = fsite[i];
  double fx, fy, fz;
  if (par[i] == i) {
    fx = fi.x; fy = fi.y; fz = fi.z;
  } else {
    const double f = fac[i];
    fx = f * fi.x; fy = f * fi.y; fz = f * fi.z;
  }
  for (int32_t k = child_start[i]; k < child_start[i + 1]; ++k) {
    const int32_t cc = child[k];
    const double g = 1.0 - fac[cc];
    const double4 fc = fsite[cc];
    fx += g * fc.x;
    fy += g * fc.y;
    fz += g * fc.z;
  }
  fatom[i] = make_double4(fx, fy, fz, 0.0);
}

void run_halgren(mdg_ctx* c, int list_id, double cutoff, double delta, double gamma,
                 int exclude) {
  const DevList& L = c->lists[list_id];
  HalgrenKArgs k;
  k.n_i = c->n_own;
  const bool reduced = (L.sites == MDG_SITES_VDW);
  k.site = reduced ? c->vsite : c->pos;
  k.vdwp = c->vdwp;
  k.vtab = c->n_vtypes ? c->vtab : nullptr;
  k.mol = c->mol;
  // the cluster kernel walks hash-built unions: its rows need no sort
  const bool want_cl = c->cluster_halgren && !c->deterministic;
  k.L = kernel_rows(c, list_id, cutoff, !want_cl);
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = cutoff * cutoff;
  k.delta = delta;
  k.gamma = gamma;
  k.force = reduced ? c->force2 : c->force;
  const bool ex = exclude && c->has_mol;
  const bool dn = k.L.dense;
#define HAL_LAUNCH(E, H)                                                              \
  if (dn) MDG_LAUNCH_SITES(c, "halgren", k.n_i, k, (k_halgren<E, H, true>));          \
  else MDG_LAUNCH_SITES(c, "halgren", k.n_i, k, (k_halgren<E, H, false>));
  if (c->deterministic) {
    if (ex) { HAL_LAUNCH(true, false) } else { HAL_LAUNCH(false, false) }
    finalize_partials(c, c->last_grid, 8, 0, 0.5);
  } else {
    MDG_CUDA_CHECK(cudaMemsetAsync(k.force, 0, (size_t)k.n_i * sizeof(double4), c->stream));
    if (dn && build_row_unions(c, list_id, k.L)) {
      const DevList::Inner& I = L.inner;
      HalgrenClArgs kc;
      kc.n_i = k.n_i;
      kc.ncl = I.ncl;
      kc.ipw = 0;
      kc.site = k.site;
      kc.vdwp = k.vdwp;
      kc.vtab = k.vtab;
      kc.uidx = I.uidx;
      kc.ucnt = I.ucnt;
      kc.ucap = I.ucap;
      kc.b = k.b;
      kc.c2 = k.c2;
      kc.delta = delta;
      kc.gamma = gamma;
      kc.force = k.force;
      kc.partials = nullptr;
      if (ex) MDG_LAUNCH_SITES(c, "halgren", kc.ncl, kc, k_halgren_cl<true>);
      else MDG_LAUNCH_SITES(c, "halgren", kc.ncl, kc, k_halgren_cl<false>);
    } else {
      if (ex) { HAL_LAUNCH(true, true) } else { HAL_LAUNCH(false, true) }
    }
    finalize_partials(c, c->last_grid, 8, 0, 1.0);
  }
#undef HAL_LAUNCH
  if (reduced) {
    MDG_LAUNCH(c, "chain_rule", grid_for(c->n_own, 256), 256, 0, k_chain_rule, c->n_own, c->force2,
               c->hpar, c->hfac, c->child_start, c->child, c->force);
  }
}

}  // namespace mdg
