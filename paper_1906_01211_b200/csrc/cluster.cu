// cluster.cu -- site clusters: the north-star "atom tiles" as molecules.
//
// A cluster is kCl = 3 consecutive sites of the sorted order. With molecules
// uploaded the order is molecule-keyed (abi.cpp mdg_topology_upload,
// resort.cu), so for water a cluster is one molecule: three sites within
// 1 A whose rows are nearly the same set.
//
// Halgren (nonpolar.cu k_halgren_cl, the default): k_row_union builds, when
// the buffered 9.5 A rows are cut again, each cluster's half union -- the
// entries past its first site of row 0, then of row 1 not in row 0, then of
// row 2 in neither -- through a per-warp shared-memory hash set, so the rows
// need no sort; the kernel then gathers j's record and adds its partner force
// once per entry for the three sites.
//
// PCG (opt-in, mdg_set_cluster_matvec): per cluster
//   U75   the sorted union of the three sites' buffered inner rows (the rows
//         cut to 7 A + 0.5 A that the field pass walks), built by
//         k_cluster_union when those rows are cut again (gated by the cut's
//         generation counter), with each row slot's position in U75 (cmap)
//         and zero pair tensors for the (site, entry) slots no row holds,
//         in 32-entry chunks (ClChunk: per site the tensors, then the indices);
//   ct    per site and entry the pair tensor (rr3, rr5), written by the field
//         pass (polar.cu k_perm_field<CLMAP>) through cmap every step: the
//         tensor within the cutoff, zero beyond.
// On config 4 U75 has 216 entries per molecule (the three 7 A rows hold 435
// pairs): the mat-vec gathers j's position and direction once per 2.0 pairs
// instead of once per pair, for 26 B of streamed index + tensors per pair
// (20 B in the per-site rows, whose stream is bound by the L1 data pipe on
// the gathers). k_tmatvec_cl is warp-specialized: a producer warp per block
// copies the chunks into the three consumer warps' stage rings (TMA bulk
// copies, full / empty mbarriers); the consumers gather and compute, lane per
// entry, the 9 sums reduced once per cluster. Measured at parity with the
// per-site stream.
//
// Reference counterpart: dipole_field_matvec_vectorized
// (proj/src/polar_vec.cpp:131-204), whose per-site gather/select of j
// (proj/src/select_impl.hpp:54-60) this replaces.
#include <climits>

#include "common.cuh"

namespace mdg {

#ifndef MDG_CL_MINB
#define MDG_CL_MINB 6
#endif

constexpr int kGrp = 4;  // lanes per cluster in the union merge (kCl used)
static_assert(kCl <= kGrp, "cluster larger than its merge group");

struct CUArgs {
  int64_t n;      // sites with rows (owned)
  int64_t ncl;    // clusters
  ListView rows;  // the rows the union covers (inner rows, ascending)
  ClChunk* __restrict__ cst;   // [ncl][nch]
  int32_t* __restrict__ ucnt;  // [ncl]
  int32_t nch, tcap;
  uint16_t* __restrict__ cmap;  // [n][rows.cap]: row slot -> union position
  const int32_t* __restrict__ gen;   // the rows' cut generation (NULL: rebuild)
  const int32_t* __restrict__ ugen;  // the generation the unions hold
};

__device__ __forceinline__ int32_t row_elem(const int4& v, int k) {
  return (k == 0) ? v.x : (k == 1) ? v.y : (k == 2) ? v.z : v.w;
}

// One warp merges 8 clusters at a time: lane 4 g + k (k < kCl) holds the
// head of row k of cluster 8 w + g; each iteration emits the group minimum
// and advances the rows whose head equals it, recording the slot's union
// position; a site whose row does not hold the entry gets a zero tensor
// there. Rows are read 4 entries per 128-bit load, the next 4 prefetched.
// Entries past tcap are counted, not stored (the host retries larger).
__global__ void __launch_bounds__(kBlock) k_cluster_union(CUArgs a) {
  if (a.gen && *a.gen == *a.ugen) return;  // the rows were not cut again
  constexpr int NG = 32 / kGrp;
  const int lane = threadIdx.x & 31;
  const int g = lane / kGrp, k = lane % kGrp;
  const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int64_t cl = warp * NG + g;
  const int64_t i = cl * kCl + k;
  const bool vc = k < kCl && cl < a.ncl;  // a site slot of the cluster's tensors
  const bool vi = vc && i < a.n;          // ... of a site with a row
  const int len = vi ? a.rows.cnt[i] : 0;
  const int4* row = reinterpret_cast<const int4*>(a.rows.nbr + (size_t)(vi ? i : 0) * a.rows.cap);
  uint16_t* map = a.cmap + (size_t)(vi ? i : 0) * a.rows.cap;
  ClChunk* cc = a.cst + (size_t)(cl < a.ncl ? cl : 0) * a.nch;
  int4 b0 = make_int4(0, 0, 0, 0), b1 = b0;
  if (len > 0) b0 = __ldcs(row);
  if (len > 4) b1 = __ldcs(row + 1);
  int h = 0;
  int32_t cur = (len > 0) ? (b0.x & 0x7fffffff) : INT_MAX;
  int s = 0;
  for (;;) {
    int32_t m = cur;
#pragma unroll
    for (int o = 1; o < kGrp; o <<= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    const bool live = m != INT_MAX;
    if (!__any_sync(0xffffffffu, live)) break;
    const bool hit = live && cur == m;
    const bool st = live && s < a.tcap;
    if (k == 0 && st) cc[s >> 5].idx[s & 31] = m;
    if (hit) map[h] = (uint16_t)min(s, 65535);
    else if (vc && st) cc[s >> 5].ten[k][s & 31] = make_double2(0.0, 0.0);
    s += live;
    h += hit;
    if (hit && (h & 3) == 0) {
      b0 = b1;
      if (h + 4 < len) b1 = __ldcs(row + (h >> 2) + 1);
    }
    const int32_t nx = row_elem(b0, h & 3) & 0x7fffffff;
    cur = hit ? ((h < len) ? nx : INT_MAX) : cur;
  }
  // pad to whole 32-entry chunks (at least one): index = the cluster's first
  // site, tensors zero, so the mat-vec computes every lane of a chunk unmasked
  if (cl < a.ncl && s <= a.tcap) {
    const int padded = max(32, (s + 31) & ~31);
    for (int e = s; e < padded; ++e) {
      if (k == 0) cc[e >> 5].idx[e & 31] = (int32_t)(cl * kCl);
      if (vc) cc[e >> 5].ten[k][e & 31] = make_double2(0.0, 0.0);
    }
  }
  if (k == 0 && cl < a.ncl) a.ucnt[cl] = s;
}

// Plain unions (no maps, no tensors) of a list's buffered rows for the
// cluster pair kernels: the merge of k_cluster_union writing the sorted
// union of each cluster's kCl rows into uidx[cl * ucap ...].
struct RUArgs {
  int64_t n, ncl;
  ListView rows;
  int32_t* __restrict__ uidx;
  int32_t* __restrict__ ucnt;
  int32_t ucap;
  const int32_t* __restrict__ gen;
  const int32_t* __restrict__ ugen;
};

// Half unions: warp per cluster; the entries past the cluster's first site
// of row 0, then those of row 1 not in row 0, then those of row 2 in neither,
// compacted by ballot and stored coalesced. The rows need no order:
// membership through a per-warp open-addressing hash set in shared memory
// (rows 0 and 1 inserted, load <= 1/2), so the cut that feeds it skips the
// row sort (kernel_rows want_sorted = false). (A sequential 3-way merge of
// sorted rows by lane groups took 2.5 ms per build on config 4, per-value
// binary search 1.4 ms, a sliding-window shuffle search 1.15 ms -- plus the
// 2.6 ms sort of the rows they needed.)
__device__ __forceinline__ uint32_t hslot(int32_t x, int tbits) {
  return ((uint32_t)x * 0x9E3779B1u) >> (32 - tbits);
}

__global__ void __launch_bounds__(kBlock) k_row_union(RUArgs a, int tbits) {
  if (a.gen && *a.gen == *a.ugen) return;  // the rows were not cut again
  extern __shared__ int32_t hmem[];
  int32_t* tab = hmem + ((size_t)(threadIdx.x >> 5) << tbits);
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t cl = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); cl < a.ncl; cl += nw) {
    const int64_t i0 = cl * kCl;
    const int nv = (int)min((int64_t)kCl, a.n - i0);
    // this cluster's table: a power of two >= 2 x the keys rows 0 and 1
    // insert (their entries past i0: counted first), within the T allocated
    // (cleared per cluster)
    int need = 0;
    for (int t = 0; t + 1 < nv; ++t) {
      const int32_t* r = a.rows.nbr + (size_t)(i0 + t) * a.rows.cap;
      const int len = a.rows.cnt[i0 + t];
      for (int b = lane; b < len; b += 32) need += (__ldg(r + b) & 0x7fffffff) > (int32_t)i0;
    }
    need = warp_allsum_i(need);
    int tb = 6;
    while (tb < tbits && (1 << tb) < 2 * need) ++tb;
    const int Tc = 1 << tb;
    __syncwarp();
    for (int e = lane; e < Tc; e += 32) tab[e] = -1;
    __syncwarp();
    int32_t* out = a.uidx + (size_t)cl * a.ucap;
    int s = 0;
    for (int t = 0; t < nv; ++t) {
      const int32_t* r = a.rows.nbr + (size_t)(i0 + t) * a.rows.cap;
      const int len = a.rows.cnt[i0 + t];
      // 4 chunks' entries loaded up front (one at a time, the loop was
      // latency-bound on them)
      for (int b4 = 0; b4 < len; b4 += 128) {
        int32_t xs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = b4 + 32 * u + lane;
          xs[u] = k < len ? (__ldg(r + k) & 0x7fffffff) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
        if (b4 + 32 * u >= len) break;  // warp-uniform
        const int32_t x = xs[u];
        bool keep = x > (int32_t)i0;
        if (keep && t > 0) {  // in an earlier row?
          for (uint32_t h = hslot(x, tb);; h = (h + 1) & (Tc - 1)) {
            const int32_t v = tab[h];
            if (v == x) {
              keep = false;
              break;
            }
            if (v < 0) break;
          }
        }
        if (keep && t + 1 < nv) {  // for the later rows' tests
          for (uint32_t h = hslot(x, tb);; h = (h + 1) & (Tc - 1))
            if (atomicCAS(&tab[h], -1, x) == -1) break;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        MDG_DASSERT(s + __popc(m) <= a.ucap);
        if (keep) out[s + __popc(m & lt)] = x;
        s += __popc(m);
        }
      }
      __syncwarp();  // this row's inserts before the next row's probes
    }
    if (lane == 0) a.ucnt[cl] = s;
  }
}

__global__ void k_cluster_gen(const int32_t* __restrict__ gen, int32_t* __restrict__ ugen) {
  *ugen = gen ? *gen : -1;
}

// E_i = sum_j rr5 (v_j . R) R - rr3 v_j at the kCl sites of each cluster over
// its entries; the PCG form writes q = p/alpha - T p and the block partial of
// p.q (as k_tmatvec_pre). The chunk padding, and sites whose row does not
// hold the entry or holds it beyond the cutoff, carry rr = 0 and contribute
// exactly 0.
//
// The stream (indices and tensors of each 32-entry chunk, and on a cluster's
// first chunk its sites' positions, directions and polarizabilities) reaches
// shared memory by bulk asynchronous copies (TMA engine, mbarrier
// transaction counts), kClStages chunks ahead of the warp; the gathers of j
// for chunk k + 1 are issued before chunk k computes. Register-level
// pipelining of the same stream was undone by the compiler's scheduling
// (ncu: long-scoreboard stalls on the loads of the chunk being computed).
//
// Minimum image: fma(-rint((x_t - x_j)/L), L, x_t - x_j), the field pass's
// wrap1 without its final t >= L/2 correction, which never fires within the
// cutoff (< L/2): the same bits for every pair with a nonzero tensor.
#ifndef MDG_CL_STAGES
#define MDG_CL_STAGES 4
#endif
constexpr int kClStages = MDG_CL_STAGES;

struct __align__(128) ClStage {
  ClChunk ch;            // the chunk: tensors per cluster site, indices
  double4 spos[kCl];     // first chunk of a cluster: its sites' positions,
  double4 sin[kCl];      // PCG directions p
  double2 spol[kCl];     // and (polarizability, ...)
};

struct ClCur {
  int32_t q;     // the warp's q-th cluster (first + q kWarps)
  int32_t base;  // first entry of the chunk
  int32_t cnt;   // the cluster's entry count
};

// Warp-specialized: warp 0 of the block is the producer -- it walks the
// chunk sequences of the three consumer warps and issues each chunk's bulk
// copy into the consumer's stage ring as soon as the consumer has released
// the stage (full / empty mbarrier pairs); warps 1-3 only wait, gather and
// compute. (With every warp issuing its own copies the kernel was
// issue-bound at ~310 instructions per chunk, most of them the copy and
// cursor bookkeeping.)
constexpr int kClConsumers = kWarps - 1;

template <bool PCG>
__global__ void __launch_bounds__(kBlock, MDG_CL_MINB) k_tmatvec_cl(CLArgs a) {
  if (PCG && a.res[27] != 0.0) return;  // converged (speculative iteration)
  __shared__ ClStage st_mem[kClConsumers][kClStages];
  __shared__ uint64_t full_mem[kClConsumers][kClStages], empty_mem[kClConsumers][kClStages];
  __shared__ double4 cs_mem[kClConsumers][3 * kCl];  // the current cluster: pos, p, polp
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc1[1] = {0.0};
  const int64_t b0 = (int64_t)blockIdx.x * a.ipw;
  const int32_t end = (int32_t)min(a.ncl, b0 + a.ipw);
  if (threadIdx.x == 0) {
    for (int c = 0; c < kClConsumers; ++c)
      for (int s = 0; s < kClStages; ++s) {
        mbar_init(&full_mem[c][s]);
        mbar_init(&empty_mem[c][s]);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // consumer c's clusters: b0 + c, b0 + c + 3, ...; a chunk = (q, base, cnt)
  auto cl_of = [&](int c, int32_t q) { return (int32_t)(b0 + c + (int64_t)q * kClConsumers); };
  auto advance = [&](int c, ClCur& u) {
    if (u.base + 32 < u.cnt) {
      u.base += 32;
      return;
    }
    ++u.q;
    u.base = 0;
    const int32_t cl = cl_of(c, u.q);
    u.cnt = cl < end ? __ldg(a.ucnt + cl) : 0;
  };
  if (w == 0) {
    // ---- producer
    ClCur u[kClConsumers];
    int k[kClConsumers];
    bool live[kClConsumers];
    for (int c = 0; c < kClConsumers; ++c) {
      const int32_t cl = cl_of(c, 0);
      live[c] = cl < end;
      u[c] = ClCur{0, 0, live[c] ? __ldg(a.ucnt + cl) : 0};
      k[c] = 0;
    }
    for (;;) {
      bool any = false;
      for (int c = 0; c < kClConsumers; ++c) {
        if (!live[c]) continue;
        any = true;
        const int s = k[c] & (kClStages - 1);
        mbar_wait(&empty_mem[c][s], ((k[c] / kClStages) & 1) ^ 1);  // the consumer released it
        if (lane == 0) {
          const int64_t cl = cl_of(c, u[c].q);
          const int64_t i0 = cl * kCl;
          const int ns = u[c].base == 0 ? (int)min((int64_t)kCl, a.n - i0) : 0;
          ClStage& S = st_mem[c][s];
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arm(&full_mem[c][s], (uint32_t)(sizeof(ClChunk) + ns * (PCG ? 80 : 32)));
          bulk_load(&S.ch, a.cst + (size_t)cl * a.nch + (u[c].base >> 5), sizeof(ClChunk),
                    &full_mem[c][s]);
          if (ns > 0) {
            bulk_load(S.spos, a.pos + i0, 32 * ns, &full_mem[c][s]);
            if (PCG) {
              bulk_load(S.sin, a.in + i0, 32 * ns, &full_mem[c][s]);
              bulk_load(S.spol, a.polp + i0, 16 * ns, &full_mem[c][s]);
            }
          }
        }
        ++k[c];
        advance(c, u[c]);
        live[c] = cl_of(c, u[c].q) < end;
      }
      if (!any) break;
    }
  } else {
    // ---- consumer c
    const int c = w - 1;
    ClStage* st = st_mem[c];
    uint64_t* full = full_mem[c];
    uint64_t* empty = empty_mem[c];
    double4* cs = cs_mem[c];
    if (cl_of(c, 0) < end) {
      ClCur cons{0, 0, __ldg(a.ucnt + cl_of(c, 0))};
      ClCur next = cons;
      advance(c, next);
      mbar_wait(&full[0], 0);
      double4 p0, m0, p1, m1;
      {
        const int32_t j = st[0].ch.idx[lane];
        p0 = ldg4(a.pos + j);
        m0 = ldg4(a.in + j);
      }
      double ex[kCl], ey[kCl], ez[kCl];
#pragma unroll
      for (int t = 0; t < kCl; ++t) ex[t] = ey[t] = ez[t] = 0.0;
      for (int kc = 0;; ++kc) {
        const int slot = kc & (kClStages - 1), nslot = (kc + 1) & (kClStages - 1);
        const bool more = cl_of(c, next.q) < end;
        if (more) {  // the next chunk's gathers, in flight during this one's math
          mbar_wait(&full[nslot], ((kc + 1) / kClStages) & 1);
          const int32_t j = st[nslot].ch.idx[lane];
          p1 = ldg4(a.pos + j);
          m1 = ldg4(a.in + j);
        }
        const ClStage& S = st[slot];
        if (cons.base == 0) {  // a new cluster: keep its site records
          if (lane < kCl) {
            cs[lane] = S.spos[lane];
            if (PCG) {
              cs[kCl + lane] = S.sin[lane];
              const double2 pp = S.spol[lane];
              cs[2 * kCl + lane] = make_double4(pp.x, pp.y, 0.0, 0.0);
            }
          }
          __syncwarp();
        }
#pragma unroll
        for (int t = 0; t < kCl; ++t) {
          const double2 r = S.ch.ten[t][lane];
          const double4 pi = cs[t];
          const double ux = __dsub_rn(pi.x, p0.x), uy = __dsub_rn(pi.y, p0.y),
                       uz = __dsub_rn(pi.z, p0.z);
          const double dx = __fma_rn(-rint(__dmul_rn(ux, a.b.ix)), a.b.lx, ux);
          const double dy = __fma_rn(-rint(__dmul_rn(uy, a.b.iy)), a.b.ly, uy);
          const double dz = __fma_rn(-rint(__dmul_rn(uz, a.b.iz)), a.b.lz, uz);
          const double dot = m0.x * dx + m0.y * dy + m0.z * dz;
          ex[t] += r.y * dot * dx - r.x * m0.x;
          ey[t] += r.y * dot * dy - r.x * m0.y;
          ez[t] += r.y * dot * dz - r.x * m0.z;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // the stage may be refilled
        if (next.q != cons.q) {  // the cluster's last chunk: reduce, write, reset
          double mx = 0, my = 0, mz = 0;  // lane t < kCl keeps site t's sums
#pragma unroll
          for (int t = 0; t < kCl; ++t) {
            const double sx = warp_allsum(ex[t]), sy = warp_allsum(ey[t]),
                         sz = warp_allsum(ez[t]);
            if (lane == t) {
              mx = sx;
              my = sy;
              mz = sz;
            }
            ex[t] = ey[t] = ez[t] = 0.0;
          }
          const int64_t i = (int64_t)cl_of(c, cons.q) * kCl + lane;
          if (lane < kCl && i < a.n) {
            if (PCG) {
              const double4 p = cs[kCl + lane];
              const double inva = 1.0 / cs[2 * kCl + lane].x;
              const double qx = p.x * inva - mx, qy = p.y * inva - my, qz = p.z * inva - mz;
              a.out[i] = make_double4(qx, qy, qz, 0.0);
              acc1[0] += p.x * qx + p.y * qy + p.z * qz;
            } else {
              a.out[i] = make_double4(mx, my, mz, 0.0);
            }
          }
          __syncwarp();
        }
        if (!more) break;
        cons = next;
        advance(c, next);
        p0 = p1;
        m0 = m1;
      }
    }
  }
  if (PCG) block_store_partials<1>(acc1, a.partials);
}

bool build_clusters(mdg_ctx* c, double cutoff, const ListView& rows, const int32_t* gen,
                    int32_t tcap, bool force) {
  PrunedList& P = c->plist;
  P.cl_valid = false;
  // (the mat-vec's minimum image relies on cutoff < L/2; union positions in 16 bits)
  if (!c->cluster_matvec || !rows.sorted || !rows.dense || !gen || c->n_own == 0 ||
      group_overlap(c) || !(2.0 * cutoff < std::min(c->lx, std::min(c->ly, c->lz))) ||
      tcap > 65504)
    return false;
  const int64_t n = c->n_own;
  const int64_t ncl = (n + kCl - 1) / kCl;
  const int32_t nch = tcap / 32;
  // rebuild unconditionally when the buffers are new / for other rows;
  // otherwise the device compares the rows' cut generation with the unions'
  const uintptr_t key[4] = {(uintptr_t)rows.nbr, (uintptr_t)rows.cap, (uintptr_t)ncl,
                            (uintptr_t)tcap};
  for (int q = 0; q < 4; ++q) force = force || !P.ubuilt || P.ukey[q] != key[q];
  const size_t need = (size_t)ncl * (size_t)nch;
  if (need > P.celems) {
    if (P.cst) cudaFree(P.cst);
    P.cst = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&P.cst, need * sizeof(ClChunk)));
    P.celems = need;
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
  const size_t mneed = (size_t)n * (size_t)rows.cap;
  if (mneed > P.melems) {
    if (P.cmap) cudaFree(P.cmap);
    P.cmap = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&P.cmap, mneed * sizeof(uint16_t)));
    P.melems = mneed;
    force = true;
  }
  CUArgs a;
  a.n = n;
  a.ncl = ncl;
  a.rows = rows;
  a.cst = P.cst;
  a.ucnt = P.ucnt;
  a.nch = nch;
  a.tcap = tcap;
  a.cmap = P.cmap;
  a.gen = force ? nullptr : gen;
  a.ugen = P.ugen;
  const int64_t warps = (ncl + 32 / kGrp - 1) / (32 / kGrp);
  const unsigned grid = (unsigned)((warps * 32 + kBlock - 1) / kBlock);
  MDG_LAUNCH(c, "cluster_union", grid, kBlock, 0, k_cluster_union, a);
  MDG_LAUNCH(c, "cluster_gen", 1, 1, 0, k_cluster_gen, gen, P.ugen);
  P.ncl = ncl;
  P.ucut = cutoff;
  P.mstride = rows.cap;
  P.tcap = tcap;
  P.nch = nch;
  for (int q = 0; q < 4; ++q) P.ukey[q] = key[q];
  P.ubuilt = true;
  return true;
}

bool build_row_unions(mdg_ctx* c, int list_id, const ListView& rows) {
  DevList& L = c->lists[list_id];
  DevList::Inner& I = L.inner;
  if (!c->cluster_halgren || c->deterministic || !rows.dense || !I.gen || c->n_own == 0)
    return false;
  const int64_t n = c->n_own;
  const int64_t ncl = (n + kCl - 1) / kCl;
  const int32_t ucap = (int32_t)std::min<int64_t>((int64_t)kCl * rows.cap, (int64_t)1 << 30);
  const uintptr_t key[3] = {(uintptr_t)rows.nbr, (uintptr_t)rows.cap, (uintptr_t)ncl};
  bool force = !I.ubuilt;
  for (int q = 0; q < 3; ++q) force = force || I.ukey[q] != key[q];
  const size_t need = (size_t)ncl * (size_t)ucap;
  if (need > I.uelems) {
    if (I.uidx) cudaFree(I.uidx);
    I.uidx = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&I.uidx, need * sizeof(int32_t)));
    I.uelems = need;
    force = true;
  }
  if (!I.ugen) {
    MDG_CUDA_CHECK(cudaMalloc(&I.ugen, sizeof(int32_t)));
    force = true;
  }
  if (ncl > I.ucnt_elems) {
    if (I.ucnt) cudaFree(I.ucnt);
    I.ucnt = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&I.ucnt, (size_t)ncl * sizeof(int32_t)));
    I.ucnt_elems = ncl;
    force = true;
  }
  RUArgs a;
  a.n = n;
  a.ncl = ncl;
  a.rows = rows;
  a.uidx = I.uidx;
  a.ucnt = I.ucnt;
  a.ucap = ucap;
  a.gen = force ? nullptr : I.gen;
  a.ugen = I.ugen;
  // hash table per warp: 2048 slots (8 KB), enough for two rows of up to
  // 1024 entries (the inserted keys) at load <= 1/2 when rows are that long
  const int tbits = 11;
  if (2 * (int64_t)L.max_cnt >= (1 << tbits)) return false;  // an empty slot always left
  const size_t smem = (size_t)kWarps * ((size_t)1 << tbits) * sizeof(int32_t);
  static size_t configured = 0;
  if (smem > configured) {
    MDG_CUDA_CHECK(cudaFuncSetAttribute(k_row_union, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    configured = smem;
  }
  const unsigned grid = (unsigned)std::min<int64_t>((ncl + kWarps - 1) / kWarps, 148 * 64);
  MDG_LAUNCH(c, "row_union", grid, kBlock, smem, k_row_union, a, tbits);
  MDG_LAUNCH(c, "cluster_gen", 1, 1, 0, k_cluster_gen, I.gen, I.ugen);
  I.ucap = ucap;
  I.ncl = ncl;
  for (int q = 0; q < 3; ++q) I.ukey[q] = key[q];
  I.ubuilt = true;
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
  k.cst = P.cst;
  k.ucnt = P.ucnt;
  k.nch = P.nch;
  k.b = make_box(c->lx, c->ly, c->lz);
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
