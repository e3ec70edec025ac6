// cluster.cu -- the PCG mat-vec on site clusters (the north-star "atom-tile"
// kernel for the solve's hot loop).
//
// A cluster is 8 consecutive sites of the spatially sorted order, i.e. a
// compact blob of ~80 A^3. Once per pruned-list build (per step, after
// k_perm_field<TPRE>) k_cluster_union merges the 8 sorted pruned rows of a
// cluster into their sorted union U_c with an 8-bit membership mask per
// entry (bit t: the pair (site 8c+t, j) is within the kernel cutoff). The
// mat-vec then walks U_c 32 entries at a time: each lane gathers ONE j's
// position and direction p_j and applies them to every site of the cluster
// whose mask bit is set -- 64 B of gathers per union entry instead of per
// directed pair (~3x fewer; the per-site kernel k_tmatvec_pre was bound by
// the L1 data pipe on those gathers, VERDICT r1 "What's weak" 2). The stored
// pair tensors (rr3, rr5) keep the per-site row layout k_perm_field<TPRE>
// writes: row i lists its pairs in ascending j, which is U_c's order
// restricted to i, so the tensor of (i = 8c+t, U_c[s]) sits at slot
// popc(bits t of U_c[0..s)) of row i -- a ballot + popc per (chunk, t), and
// the active lanes of one t read consecutive tensors (coalesced).
//
// The pair vector R = r_i - r_j is formed as o_t + d0_j with
// d0_j = minimum_image(r_anchor - r_j) once per union entry and
// o_t = minimum_image(r_i - r_anchor) once per cluster (3 adds per pair
// instead of a minimum image); this is the same vector as the per-pair
// minimum image whenever |o_t| + cutoff < L/2 on every axis, which
// k_cluster_union checks per cluster ("wide" clusters use the per-pair
// minimum image). The pair SET is the pruned rows', selected bit-exactly by
// the reference predicate in k_perm_field; only the last bits of R differ
// (rounding of o_t + d0_j), far below the solver tolerance.
//
// Reference counterpart: dipole_field_matvec_vectorized
// (proj/src/polar_vec.cpp:131-204), whose per-site gather/select of j
// (proj/src/select_impl.hpp:54-60) this replaces.
#include <climits>

#include "common.cuh"

namespace mdg {

#ifndef MDG_CL_MINB
#define MDG_CL_MINB 1
#endif
#if MDG_CL_MINB > 1
#define MDG_CL_BOUNDS __launch_bounds__(kBlock, MDG_CL_MINB)
#else
#define MDG_CL_BOUNDS __launch_bounds__(kBlock)
#endif

struct CUArgs {
  int64_t n;      // sites with rows (owned)
  int64_t ncl;    // clusters
  const int32_t* __restrict__ pnbr;
  const int32_t* __restrict__ pcnt;
  int32_t pcap;
  const double4* __restrict__ pos;
  Box b;
  double cutoff;
  uint32_t* __restrict__ ucl;  // [ncl][ucap]: j | mask << 24
  int32_t* __restrict__ ucnt;  // [ncl]: entries | wide << 31
  int32_t ucap;
};

__device__ __forceinline__ int32_t row_elem(const int4& v, int k) {
  return (k == 0) ? v.x : (k == 1) ? v.y : (k == 2) ? v.z : v.w;
}

// One warp merges 32/G clusters at a time: lane G g + k holds the head of row
// k of cluster (32/G) w + g; each iteration emits the group minimum with the
// mask of the rows whose head equals it and advances those rows. Rows are
// read 4 entries per 128-bit load, the next 4 prefetched.
template <int G>
__global__ void __launch_bounds__(kBlock) k_cluster_union(CUArgs a) {
  constexpr int NG = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane / G, k = lane % G;
  const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int64_t cl = warp * NG + g;
  const int64_t i = cl * G + k;
  const bool vi = cl < a.ncl && i < a.n;
  const int len = vi ? a.pcnt[i] : 0;
  const int4* row = reinterpret_cast<const int4*>(a.pnbr + (size_t)(vi ? i : 0) * a.pcap);
  int4 b0 = make_int4(0, 0, 0, 0), b1 = b0;
  if (len > 0) b0 = __ldcs(row);
  if (len > 4) b1 = __ldcs(row + 1);
  int h = 0;
  int32_t cur = (len > 0) ? (b0.x & 0x7fffffff) : INT_MAX;
  // wide-cluster test: max |o_t| component + cutoff against the half box
  double om = 0.0;
  if (vi) {
    const double4 pi = a.pos[i], pa = a.pos[cl * G];
    double ox, oy, oz;
    min_image(a.b, pi.x, pi.y, pi.z, pa.x, pa.y, pa.z, ox, oy, oz);
    om = fmax(fabs(ox), fmax(fabs(oy), fabs(oz)));
  }
#pragma unroll
  for (int o = 1; o < G; o <<= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
  uint32_t* out = a.ucl + (size_t)(cl < a.ncl ? cl : 0) * a.ucap;
  int s = 0;
  for (;;) {
    int32_t m = cur;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    const bool live = m != INT_MAX;
    if (!__any_sync(0xffffffffu, live)) break;
    const bool hit = live && cur == m;
    const unsigned bm = (__ballot_sync(0xffffffffu, hit) >> (G * g)) & ((1u << G) - 1u);
    MDG_DASSERT(!live || s < a.ucap);
    if (k == 0 && live) out[s] = (uint32_t)m | (bm << 24);
    s += live;
    h += hit;
    if (hit && (h & 3) == 0) {
      b0 = b1;
      if (h + 4 < len) b1 = __ldcs(row + (h >> 2) + 1);
    }
    const int32_t nx = row_elem(b0, h & 3) & 0x7fffffff;
    cur = hit ? ((h < len) ? nx : INT_MAX) : cur;
  }
  if (k == 0 && cl < a.ncl) {
    const double hmin = fmin(a.b.hx, fmin(a.b.hy, a.b.hz));
    const bool wide = !(om + a.cutoff + 1e-6 < hmin);
    a.ucnt[cl] = s | (wide ? (int32_t)0x80000000 : 0);
  }
}

// E_i = sum_j rr5 (v_j . R) R - rr3 v_j over the cluster's union; the PCG
// form writes q = p/alpha - T p and the block partial of p.q (as
// k_tmatvec_pre). Software-pipelined: the union entries of chunk c+2, the
// gathers of j and the pair-tensor loads of chunk c+1 are in flight while
// chunk c is computed.
template <int G, bool PCG>
__global__ void MDG_CL_BOUNDS k_tmatvec_cl(CLArgs a) {
  if (PCG && a.res[27] != 0.0) return;  // converged (speculative iteration)
  __shared__ double4 s_o[kWarps][G];  // o_t (minimum image r_i - r_anchor)
  __shared__ double4 s_p[kWarps][G];  // r_i (wide clusters)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  double acc1[1] = {0.0};
  MDG_SITE_LOOP(cl, a.ncl, a.ipw) {
    const int64_t anchor = cl * G;
    const double4 pa = a.pos[anchor];
    if (lane < G) {
      const int64_t i = anchor + lane;
      double4 pi = pa;
      if (i < a.n) pi = a.pos[i];
      double ox, oy, oz;
      min_image(a.b, pi.x, pi.y, pi.z, pa.x, pa.y, pa.z, ox, oy, oz);
      s_o[w][lane] = make_double4(ox, oy, oz, 0.0);
      s_p[w][lane] = pi;
    }
    __syncwarp();
    const int32_t craw = a.ucnt[cl];
    const bool wide = craw < 0;
    const int ucount = craw & 0x7fffffff;
    MDG_DASSERT(ucount <= a.ucap);
    const uint32_t* urow = a.ucl + (size_t)cl * a.ucap;
    const double2* tp[G];
    double ex[G], ey[G], ez[G];
#pragma unroll
    for (int t = 0; t < G; ++t) {
      tp[t] = a.trr + (size_t)(anchor + t) * a.pcap;
      ex[t] = ey[t] = ez[t] = 0.0;
    }
    // pipeline fill: u of chunks 0 and 1, gathers + tensors of chunk 0
    uint32_t u0 = (lane < ucount) ? __ldcs(urow + lane) : 0u;
    uint32_t u1 = (32 + lane < ucount) ? __ldcs(urow + 32 + lane) : 0u;
    double4 pj = ldg4(a.pos + (u0 & 0xffffffu));
    double4 mj = ldg4(a.in + (u0 & 0xffffffu));
    double2 rr[G];
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const bool bit = (u0 >> (24 + t)) & 1u;
      const unsigned bm = __ballot_sync(0xffffffffu, bit);
      rr[t] = bit ? __ldcs(tp[t] + __popc(bm & lt)) : make_double2(0.0, 0.0);
      tp[t] += __popc(bm);
    }
    for (int s0 = 0; s0 < ucount; s0 += 32) {
      // chunk c+1: gathers and tensors; chunk c+2: union entries
      const uint32_t u2 = (s0 + 64 + lane < ucount) ? __ldcs(urow + s0 + 64 + lane) : 0u;
      const double4 pjn = ldg4(a.pos + (u1 & 0xffffffu));
      const double4 mjn = ldg4(a.in + (u1 & 0xffffffu));
      double2 rrn[G];
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const bool bit = (u1 >> (24 + t)) & 1u;
        const unsigned bm = __ballot_sync(0xffffffffu, bit);
        rrn[t] = bit ? __ldcs(tp[t] + __popc(bm & lt)) : make_double2(0.0, 0.0);
        tp[t] += __popc(bm);
      }
      // chunk c
      if (!wide) {
        double d0x, d0y, d0z;
        min_image(a.b, pa.x, pa.y, pa.z, pj.x, pj.y, pj.z, d0x, d0y, d0z);
#pragma unroll
        for (int t = 0; t < G; ++t) {
          const double4 o = s_o[w][t];
          const double dx = o.x + d0x, dy = o.y + d0y, dz = o.z + d0z;
          const double dot = mj.x * dx + mj.y * dy + mj.z * dz;
          const double t5 = rr[t].y * dot;
          ex[t] += t5 * dx - rr[t].x * mj.x;
          ey[t] += t5 * dy - rr[t].x * mj.y;
          ez[t] += t5 * dz - rr[t].x * mj.z;
        }
      } else {
#pragma unroll
        for (int t = 0; t < G; ++t) {
          const double4 pi = s_p[w][t];
          double dx, dy, dz;
          min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz);
          const double dot = mj.x * dx + mj.y * dy + mj.z * dz;
          const double t5 = rr[t].y * dot;
          ex[t] += t5 * dx - rr[t].x * mj.x;
          ey[t] += t5 * dy - rr[t].x * mj.y;
          ez[t] += t5 * dz - rr[t].x * mj.z;
        }
      }
      pj = pjn;
      mj = mjn;
#pragma unroll
      for (int t = 0; t < G; ++t) rr[t] = rrn[t];
      u1 = u2;
    }
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const double sx = warp_allsum(ex[t]), sy = warp_allsum(ey[t]), sz = warp_allsum(ez[t]);
      const int64_t i = anchor + t;
      if (lane == t && i < a.n) {
        if (PCG) {
          const double4 p = a.in[i];
          const double inva = 1.0 / a.polp[i].x;
          const double qx = p.x * inva - sx, qy = p.y * inva - sy, qz = p.z * inva - sz;
          a.out[i] = make_double4(qx, qy, qz, 0.0);
          acc1[0] += p.x * qx + p.y * qy + p.z * qz;
        } else {
          a.out[i] = make_double4(sx, sy, sz, 0.0);
        }
      }
    }
    __syncwarp();
  }
  if (PCG) block_store_partials<1>(acc1, a.partials);
}

static int cl_sites() {
  static const int g = env_int("MDG_CL_SITES", 4) == 8 ? 8 : 4;
  return g;
}

bool build_clusters(mdg_ctx* c, double cutoff) {
  PrunedList& P = c->plist;
  P.cl_valid = false;
  static const int enabled = env_int("MDG_CLUSTER_MATVEC", 0);  // opt-in: measured slower (DESIGN 4)
  if (!enabled || !P.valid || !P.sorted || c->n >= (1 << 24) || c->n_own == 0) return false;
  const int64_t n = c->n_own;
  const int G = cl_sites();
  const int64_t ncl = (n + G - 1) / G;
  // the union of G rows is at most their total length
  const int32_t ucap = (int32_t)std::min<int64_t>((int64_t)G * P.cap, (int64_t)1 << 30);
  const size_t need = (size_t)ncl * (size_t)ucap;
  if (need > P.uelems) {
    if (P.ucl) cudaFree(P.ucl);
    P.ucl = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&P.ucl, need * sizeof(uint32_t)));
    P.uelems = need;
  }
  if (ncl > P.ucnt_elems) {
    if (P.ucnt) cudaFree(P.ucnt);
    P.ucnt = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&P.ucnt, (size_t)ncl * sizeof(int32_t)));
    P.ucnt_elems = ncl;
  }
  CUArgs a;
  a.n = n;
  a.ncl = ncl;
  a.pnbr = P.nbr;
  a.pcnt = P.cnt;
  a.pcap = P.cap;
  a.pos = c->pos;
  a.b = make_box(c->lx, c->ly, c->lz);
  a.cutoff = cutoff;
  a.ucl = P.ucl;
  a.ucnt = P.ucnt;
  a.ucap = ucap;
  const int64_t warps = (ncl + 32 / G - 1) / (32 / G);
  const unsigned grid = (unsigned)((warps * 32 + kBlock - 1) / kBlock);
  if (G == 8) MDG_LAUNCH(c, "cluster_union", grid, kBlock, 0, k_cluster_union<8>, a);
  else MDG_LAUNCH(c, "cluster_union", grid, kBlock, 0, k_cluster_union<4>, a);
  P.ucap = ucap;
  P.ncl = ncl;
  P.cl_valid = true;
  return true;
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
  k.in = in;
  k.out = out;
  k.partials = c->partials;
  k.res = c->results;
  return k;
}

const void* cl_matvec_kernel(bool pcg) {
  if (cl_sites() == 8)
    return pcg ? (const void*)k_tmatvec_cl<8, true> : (const void*)k_tmatvec_cl<8, false>;
  return pcg ? (const void*)k_tmatvec_cl<4, true> : (const void*)k_tmatvec_cl<4, false>;
}

void cl_matvec_launch(mdg_ctx* c, CLArgs& k, bool pcg, const char* name) {
  if (cl_sites() == 8) {
    if (pcg) MDG_LAUNCH_SITES(c, name, k.ncl, k, (k_tmatvec_cl<8, true>));
    else MDG_LAUNCH_SITES(c, name, k.ncl, k, (k_tmatvec_cl<8, false>));
  } else {
    if (pcg) MDG_LAUNCH_SITES(c, name, k.ncl, k, (k_tmatvec_cl<4, true>));
    else MDG_LAUNCH_SITES(c, name, k.ncl, k, (k_tmatvec_cl<4, false>));
  }
}

// raw launch for graph capture (grid and partials fixed by the caller)
void cl_matvec_launch_raw(const CLArgs& k, unsigned grid, cudaStream_t s) {
  if (cl_sites() == 8) k_tmatvec_cl<8, true><<<grid, kBlock, 0, s>>>(k);
  else k_tmatvec_cl<4, true><<<grid, kBlock, 0, s>>>(k);
}

}  // namespace mdg
