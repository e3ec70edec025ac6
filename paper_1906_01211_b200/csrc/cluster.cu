// cluster.cu -- the PCG mat-vec on site clusters (the north-star "atom-tile"
// kernel for the solve's hot loop).
//
// A cluster is 4 consecutive sites of the spatially sorted order (a compact
// blob of ~40 A^3). Its union list U_c is the sorted union of the 4 sites'
// buffered inner rows (the rows cut to 7 A + 0.5 A that k_perm_field<TPRE>
// walks), built when those rows are cut again -- on the device, gated by the
// cut's own flag, so in the static benchmark once per list rebuild and in
// dynamics once per re-cut -- by k_cluster_union.
//
// The mat-vec maps a warp onto 8 union entries x 4 cluster sites per step:
// lane 4s + t handles the pair (site t, U_c[s]). The 4 lanes of an entry load
// the same j, so one warp-wide gather touches 8 records instead of 32
// (~3x fewer L1 wavefronts per pair than the per-site stream, which is bound
// by the L1 data pipe on those gathers). Each lane tests its pair with the
// reference predicate, op for op the one k_perm_field used to build the
// pruned rows (same minimum image of the same operands, same cutoff^2), so the
// in-range pairs of site t are exactly its pruned row, in the same (ascending
// j) order; the pair tensor is read at rank popc(ballot & earlier lanes of
// the same t) past the row's running base. A lane accumulates the field of
// its own site t only (3 doubles); the lanes of a site are summed once per
// cluster (xor 4, 8, 16).
//
// Reference counterpart: dipole_field_matvec_vectorized
// (proj/src/polar_vec.cpp:131-204), whose per-site gather/select of j
// (proj/src/select_impl.hpp:54-60) this replaces.
#include <climits>

#include "common.cuh"

namespace mdg {

#ifndef MDG_CL_MINB
#define MDG_CL_MINB 4
#endif

constexpr int kCl = 4;  // sites per cluster

struct CUArgs {
  int64_t n;      // sites with rows (owned)
  int64_t ncl;    // clusters
  ListView rows;  // the rows the union covers (inner rows, ascending)
  int32_t* __restrict__ ucl;  // [ncl][ucap]
  int32_t* __restrict__ ucnt;  // [ncl]
  int32_t ucap;
  const int32_t* __restrict__ gen;   // the rows' cut generation (NULL: rebuild)
  const int32_t* __restrict__ ugen;  // the generation the unions hold
};

__device__ __forceinline__ int32_t row_elem(const int4& v, int k) {
  return (k == 0) ? v.x : (k == 1) ? v.y : (k == 2) ? v.z : v.w;
}

// One warp merges 8 clusters at a time: lane 4 g + k holds the head of row k
// of cluster 8 w + g; each iteration emits the group minimum and advances
// the rows whose head equals it. Rows are read 4 entries per 128-bit load,
// the next 4 prefetched.
__global__ void __launch_bounds__(kBlock) k_cluster_union(CUArgs a) {
  if (a.gen && *a.gen == *a.ugen) return;  // the rows were not cut again
  constexpr int NG = 32 / kCl;
  const int lane = threadIdx.x & 31;
  const int g = lane / kCl, k = lane % kCl;
  const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int64_t cl = warp * NG + g;
  const int64_t i = cl * kCl + k;
  const bool vi = cl < a.ncl && i < a.n;
  const int len = vi ? a.rows.cnt[i] : 0;
  const int4* row = reinterpret_cast<const int4*>(a.rows.nbr + (size_t)(vi ? i : 0) * a.rows.cap);
  int4 b0 = make_int4(0, 0, 0, 0), b1 = b0;
  if (len > 0) b0 = __ldcs(row);
  if (len > 4) b1 = __ldcs(row + 1);
  int h = 0;
  int32_t cur = (len > 0) ? (b0.x & 0x7fffffff) : INT_MAX;
  int32_t* out = a.ucl + (size_t)(cl < a.ncl ? cl : 0) * a.ucap;
  int s = 0;
  for (;;) {
    int32_t m = cur;
#pragma unroll
    for (int o = 1; o < kCl; o <<= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    const bool live = m != INT_MAX;
    if (!__any_sync(0xffffffffu, live)) break;
    const bool hit = live && cur == m;
    MDG_DASSERT(!live || s < a.ucap);
    if (k == 0 && live) out[s] = m;
    s += live;
    h += hit;
    if (hit && (h & 3) == 0) {
      b0 = b1;
      if (h + 4 < len) b1 = __ldcs(row + (h >> 2) + 1);
    }
    const int32_t nx = row_elem(b0, h & 3) & 0x7fffffff;
    cur = hit ? ((h < len) ? nx : INT_MAX) : cur;
  }
  if (k == 0 && cl < a.ncl) a.ucnt[cl] = s;
}

__global__ void k_cluster_gen(const int32_t* __restrict__ gen, int32_t* __restrict__ ugen) {
  *ugen = gen ? *gen : -1;
}

// E_i = sum_j rr5 (v_j . R) R - rr3 v_j over the cluster's union; the PCG
// form writes q = p/alpha - T p and the block partial of p.q (as
// k_tmatvec_pre).
template <bool PCG>
__global__ void __launch_bounds__(kBlock, MDG_CL_MINB) k_tmatvec_cl(CLArgs a) {
  if (PCG && a.res[27] != 0.0) return;  // converged (speculative iteration)
  const int lane = threadIdx.x & 31;
  const int t = lane & (kCl - 1), sl = lane / kCl;
  const unsigned same_t = 0x11111111u << t;
  const unsigned earlier = lanemask_lt() & same_t;
  double acc1[1] = {0.0};
  MDG_SITE_LOOP(cl, a.ncl, a.ipw) {
    const int64_t i = cl * kCl + t;
    const bool vi = i < a.n;
    const double4 pi = a.pos[vi ? i : cl * kCl];
    const int ucount = a.ucnt[cl];
    MDG_DASSERT(ucount >= 0 && ucount <= a.ucap);
    const int32_t* urow = a.ucl + (size_t)cl * a.ucap;
    const double2* trow = a.trr + (size_t)(vi ? i : 0) * a.pcap;
    int base = 0;
    double ex = 0, ey = 0, ez = 0;
    for (int s0 = 0; s0 < ucount; s0 += 32 / kCl) {
      const int s = s0 + sl;
      const bool vs = s < ucount;
      const int32_t j = vs ? __ldg(urow + s) : (int32_t)(cl * kCl);
      const double4 pj = ldg4(a.pos + j);
      const double4 mj = ldg4(a.in + j);
      double dx, dy, dz;
      // the pruned rows' predicate (k_perm_field): same operands, same ops
      const double r2 = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
      const bool in = vs && vi && j != (int32_t)i && r2 <= a.c2;
      const unsigned bm = __ballot_sync(0xffffffffu, in);
      double2 rr = make_double2(0.0, 0.0);
      if (in) rr = __ldcs(trow + base + __popc(bm & earlier));
      base += __popc(bm & same_t);
      const double dot = mj.x * dx + mj.y * dy + mj.z * dz;
      const double t5 = rr.y * dot;
      ex += t5 * dx - rr.x * mj.x;
      ey += t5 * dy - rr.x * mj.y;
      ez += t5 * dz - rr.x * mj.z;
    }
#pragma unroll
    for (int o = kCl; o < 32; o <<= 1) {
      ex += __shfl_xor_sync(0xffffffffu, ex, o);
      ey += __shfl_xor_sync(0xffffffffu, ey, o);
      ez += __shfl_xor_sync(0xffffffffu, ez, o);
    }
    if (lane < kCl && vi) {
      MDG_DASSERT(base <= a.pcap);
      if (PCG) {
        const double4 p = a.in[i];
        const double inva = 1.0 / a.polp[i].x;
        const double qx = p.x * inva - ex, qy = p.y * inva - ey, qz = p.z * inva - ez;
        a.out[i] = make_double4(qx, qy, qz, 0.0);
        acc1[0] += p.x * qx + p.y * qy + p.z * qz;
      } else {
        a.out[i] = make_double4(ex, ey, ez, 0.0);
      }
    }
  }
  if (PCG) block_store_partials<1>(acc1, a.partials);
}

void build_clusters(mdg_ctx* c, double cutoff, const ListView& rows, const int32_t* gen) {
  PrunedList& P = c->plist;
  static const int enabled = env_int("MDG_CLUSTER_MATVEC", 0);  // opt-in: measured slower (DESIGN 4)
  if (!enabled || !P.valid || !P.sorted || !rows.sorted || !rows.dense || !gen ||
      c->n_own == 0) {
    P.cl_valid = false;
    return;
  }
  const int64_t n = c->n_own;
  const int64_t ncl = (n + kCl - 1) / kCl;
  // the union of kCl rows is at most their total length
  const int32_t ucap = (int32_t)std::min<int64_t>((int64_t)kCl * rows.cap, (int64_t)1 << 30);
  // rebuild unconditionally when the union buffer is new / for other rows;
  // otherwise the device compares the rows' cut generation with the unions'
  const uintptr_t key[3] = {(uintptr_t)rows.nbr, (uintptr_t)rows.cap, (uintptr_t)ncl};
  bool force = !P.ubuilt || P.ukey[0] != key[0] || P.ukey[1] != key[1] || P.ukey[2] != key[2];
  const size_t need = (size_t)ncl * (size_t)ucap;
  if (need > P.uelems) {
    if (P.ucl) cudaFree(P.ucl);
    P.ucl = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&P.ucl, need * sizeof(int32_t)));
    P.uelems = need;
    force = true;
  }
  if (!P.ugen) {
    MDG_CUDA_CHECK(cudaMalloc(&P.ugen, sizeof(int32_t)));
    force = true;
  }
  if (ncl > P.ucnt_elems) {
    if (P.ucnt) cudaFree(P.ucnt);
    P.ucnt = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&P.ucnt, (size_t)ncl * sizeof(int32_t)));
    P.ucnt_elems = ncl;
    force = true;
  }
  CUArgs a;
  a.n = n;
  a.ncl = ncl;
  a.rows = rows;
  a.ucl = P.ucl;
  a.ucnt = P.ucnt;
  a.ucap = ucap;
  a.gen = force ? nullptr : gen;
  a.ugen = P.ugen;
  const int64_t warps = (ncl + 32 / kCl - 1) / (32 / kCl);
  const unsigned grid = (unsigned)((warps * 32 + kBlock - 1) / kBlock);
  MDG_LAUNCH(c, "cluster_union", grid, kBlock, 0, k_cluster_union, a);
  MDG_LAUNCH(c, "cluster_gen", 1, 1, 0, k_cluster_gen, gen, P.ugen);
  P.ucap = ucap;
  P.ncl = ncl;
  P.ucut = cutoff;
  for (int q = 0; q < 3; ++q) P.ukey[q] = key[q];
  P.ubuilt = true;
  P.cl_valid = true;
}

CLArgs cl_args(mdg_ctx* c, const double4* in, double4* out) {
  const PrunedList& P = c->plist;
  CLArgs k;
  k.n = c->n_own;
  k.ncl = P.ncl;
  k.ipw = 0;
  k.pos = c->pos;
  k.polp = c->polp;
  k.ucl = P.ucl;
  k.ucnt = P.ucnt;
  k.ucap = P.ucap;
  k.trr = P.trr;
  k.pcap = P.cap;
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = P.ucut * P.ucut;  // as k_perm_field's c2
  k.in = in;
  k.out = out;
  k.partials = c->partials;
  k.res = c->results;
  return k;
}

const void* cl_matvec_kernel(bool pcg) {
  return pcg ? (const void*)k_tmatvec_cl<true> : (const void*)k_tmatvec_cl<false>;
}

void cl_matvec_launch(mdg_ctx* c, CLArgs& k, bool pcg, const char* name) {
  if (pcg) MDG_LAUNCH_SITES(c, name, k.ncl, k, k_tmatvec_cl<true>);
  else MDG_LAUNCH_SITES(c, name, k.ncl, k, k_tmatvec_cl<false>);
}

// raw launch for graph capture (grid and partials fixed by the caller)
void cl_matvec_launch_raw(const CLArgs& k, unsigned grid, cudaStream_t s) {
  k_tmatvec_cl<true><<<grid, kBlock, 0, s>>>(k);
}

}  // namespace mdg
