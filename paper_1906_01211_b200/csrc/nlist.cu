// nlist.cu -- neighbour-list construction on the device.
//
// Replaces build_cell_grid + build_neighbor_table
// (proj/src/neighbors.cpp:10-36, proj/src/neighbors_vec.cpp:8-94).
// 1. cell id per site (grid nc = max(1, floor(L / cutoff)) per axis, as the
//    reference), counting sort of site ids into cells (histogram, scan,
//    scatter, then a per-cell sort so the order is deterministic);
// 2. one thread per site sweeps the deduplicated 27-cell stencil and keeps
//    every j != i with dist2(wrap1(r_i - r_j)) <= cutoff^2 -- the exact
//    reference predicate, so the pair SET is bit-identical;
// 3. output is a FULL list (both directions) in sliced-ELL layout so the pair
//    kernels need no j-side scatter (no atomics) and read indices coalesced.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace mdg {

__global__ void k_cell_assign(int64_t n, const double4* __restrict__ P, Grid g,
                              int32_t* __restrict__ cell_of, int32_t* __restrict__ count) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = P[i];
  // proj/src/neighbors.cpp:28-30
  const int cx = min(g.ncx - 1, (int)(p.x / g.ex));
  const int cy = min(g.ncy - 1, (int)(p.y / g.ey));
  const int cz = min(g.ncz - 1, (int)(p.z / g.ez));
  const int c = (cx * g.ncy + cy) * g.ncz + cz;
  cell_of[i] = c;
  atomicAdd(&count[c], 1);
}

// Exclusive scan of count[0..m) into start[0..m]; one block of 1024 threads,
// each owning a contiguous chunk (m is at most a few 10^5 cells).
__global__ void k_scan(int64_t m, const int32_t* count, int32_t* __restrict__ start,
                       int32_t* fill) {
  __shared__ int32_t sums[1024];
  const int t = threadIdx.x;
  const int64_t chunk = (m + 1023) / 1024;
  const int64_t b = t * chunk, e = min(m, b + chunk);
  int32_t s = 0;
  for (int64_t k = b; k < e; ++k) s += count[k];
  sums[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    int32_t v = (t >= o) ? sums[t - o] : 0;
    __syncthreads();
    sums[t] += v;
    __syncthreads();
  }
  int32_t run = sums[t] - s;
  for (int64_t k = b; k < e; ++k) {
    const int32_t v = count[k];  // count may alias fill
    start[k] = run;
    fill[k] = run;
    run += v;
  }
  if (t == 1023) start[m] = sums[1023];
}

__global__ void k_cell_fill(int64_t n, const int32_t* __restrict__ cell_of,
                            int32_t* __restrict__ fill, int32_t* __restrict__ atoms) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t slot = atomicAdd(&fill[cell_of[i]], 1);
  atoms[slot] = (int32_t)i;
}

// insertion sort of each cell's ids (cells hold O(100) sites)
__global__ void k_cell_sort(int64_t m, const int32_t* __restrict__ start,
                            int32_t* __restrict__ atoms) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= m) return;
  const int32_t b = start[c], e = start[c + 1];
  for (int32_t k = b + 1; k < e; ++k) {
    const int32_t v = atoms[k];
    int32_t q = k - 1;
    while (q >= b && atoms[q] > v) {
      atoms[q + 1] = atoms[q];
      --q;
    }
    atoms[q + 1] = v;
  }
}

// Cells have edge >= cutoff / kReach, so every partner is within kReach cells
// per axis. x, y: the deduplicated periodic cells c-kReach .. c+kReach; z: the
// same cells as at most two contiguous runs, each one contiguous range of the
// cell-sorted site array (cells are numbered z-fastest).
constexpr int kReach = 2;
constexpr int kSpan = 2 * kReach + 1;

__device__ __forceinline__ int axis_cells(int c, int nc, int (&out)[kSpan]) {
  if (kSpan >= nc) {
    for (int k = 0; k < nc; ++k) out[k] = k;
    return nc;
  }
  for (int d = -kReach; d <= kReach; ++d) out[d + kReach] = (c + d + nc) % nc;
  return kSpan;
}

__device__ __forceinline__ int axis_runs(int c, int nc, int (&lo)[2], int (&hi)[2]) {
  if (kSpan >= nc) { lo[0] = 0; hi[0] = nc - 1; return 1; }
  const int a = c - kReach, b = c + kReach;
  if (a < 0) { lo[0] = 0; hi[0] = b; lo[1] = a + nc; hi[1] = nc - 1; return 2; }
  if (b >= nc) { lo[0] = a; hi[0] = nc - 1; lo[1] = 0; hi[1] = b - nc; return 2; }
  lo[0] = a; hi[0] = b;
  return 1;
}

// Warp per site: lanes sweep a cell's sites 32 at a time (coalesced cell
// reads), a ballot compacts the hits, and the row is written contiguously
// (full 128-B lines), so the 2-4 GB list costs one pass of HBM writes.
__global__ void __launch_bounds__(kBlock) k_nlist_build(
    int64_t n_i, int ipw, const double4* __restrict__ P, const int32_t* __restrict__ cell_of,
    Grid g, const int32_t* __restrict__ start, const int32_t* __restrict__ atoms, Box b,
    double c2, int32_t cap, int32_t* __restrict__ nbr, int32_t* __restrict__ cnt,
    const int32_t* __restrict__ perm, int32_t* __restrict__ flag) {
  // per warp: the site's candidate runs (contiguous ranges of the cell-sorted
  // site array) and their exclusive prefix lengths
  constexpr int kMaxRuns = kSpan * kSpan * 2;  // <= 64: two per lane
  static_assert(kMaxRuns <= 64, "candidate runs: two per lane");
  __shared__ int32_t run_s[kWarps][64], run_p[kWarps][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* rs = run_s[warp];
  int32_t* rp = run_p[warp];
  MDG_SITE_LOOP(i, n_i, ipw) {
    const double4 pi = P[i];
    const int c = cell_of[i];
    const int cz = c % g.ncz, cy = (c / g.ncz) % g.ncy, cx = c / (g.ncz * g.ncy);
    int xs[kSpan], ys[kSpan], zlo[2], zhi[2];
    const int nx = axis_cells(cx, g.ncx, xs), ny = axis_cells(cy, g.ncy, ys),
              nz = axis_runs(cz, g.ncz, zlo, zhi);
    const int nruns = nx * ny * nz;
    // runs in the same (x, y, z-run) order as the cell walk; lane r takes run
    // r and r + 32, then a warp scan of the lengths
    int len0 = 0, len1 = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      int len = 0;
      if (r < nruns) {
        const int q = r % nz, ab = r / nz;
        const int col = (xs[ab / ny] * g.ncy + ys[ab % ny]) * g.ncz;
        const int32_t s0 = start[col + zlo[q]];
        rs[r] = s0;
        len = start[col + zhi[q] + 1] - s0;
      }
      if (h == 0) len0 = len; else len1 = len;
    }
    int inc0 = len0, inc1 = len1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(0xffffffffu, inc0, o);
      const int t1 = __shfl_up_sync(0xffffffffu, inc1, o);
      if (lane >= o) { inc0 += t0; inc1 += t1; }
    }
    const int tot0 = __shfl_sync(0xffffffffu, inc0, 31);
    rp[lane] = inc0 - len0;
    rp[lane + 32] = tot0 + inc1 - len1;
    const int total = tot0 + __shfl_sync(0xffffffffu, inc1, 31);
    __syncwarp();
    // virtual candidate index v -> site-array slot (run by binary search)
    auto slot_of = [&](int v) {
      int lo = 0, hi = nruns - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rp[mid] <= v) lo = mid; else hi = mid - 1;
      }
      return rs[lo] + (v - rp[lo]);
    };
    int32_t* out = nbr + (size_t)i * (size_t)cap;
    int32_t k = 0;  // warp-uniform row length
    // software pipeline: candidate indices one chunk ahead of the test
    int32_t ja = (lane < total) ? __ldg(atoms + slot_of(lane)) : (int32_t)i;
    for (int base = 0; base < total; base += 32) {
      const int vn = base + 32 + lane;
      const int32_t jb = (vn < total) ? __ldg(atoms + slot_of(vn)) : (int32_t)i;
      bool in = false;
      if (ja != (int32_t)i) {
        const double4 pj = ldg4(P + ja);
        double dx, dy, dz;
        in = min_image(b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz) <= c2;
      }
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (in) {
        const int32_t pos = k + __popc(m & lanemask_lt());
        if (pos < cap) out[pos] = ja;
      }
      k += __popc(m);
      ja = jb;
    }
    __syncwarp();
    if (lane == 0) cnt[i] = k;
    // reference capacity rule: the half list stores a pair on the lower
    // caller index and caps it at kMaxNeighbors (proj/src/neighbors_vec.cpp:80-83).
    // Only a row longer than the cap can break it: count its upper pairs.
    if (k > MDG_MAX_NEIGHBORS && k <= cap) {
      const int32_t oi = perm[i];
      int32_t upper = 0;
      for (int e = lane; e < k; e += 32) upper += (__ldg(perm + out[e]) > oi) ? 1 : 0;
      upper = warp_allsum_i(upper);
      if (lane == 0 && upper > MDG_MAX_NEIGHBORS) atomicMin(&flag[0], oi);
    }  // (k > cap: the host retries with the true maximum, then counts)
  }
}

// Cell-per-warp build: every site of a cell has the same candidate runs, so
// one warp walks them once for up to 32 of the cell's owned sites at a time
// (site q of the group keeps its row length in lane q): each candidate's id
// and position are loaded once per group instead of once per site. Rows are
// identical to k_nlist_build's (same candidate order).
__global__ void __launch_bounds__(kBlock) k_nlist_cells(
    int64_t ncell, int64_t n_own, const double4* __restrict__ P, Grid g,
    const int32_t* __restrict__ start, const int32_t* __restrict__ atoms, Box b, double c2,
    int32_t cap, int32_t* __restrict__ nbr, int32_t* __restrict__ cnt,
    const int32_t* __restrict__ perm, int32_t* __restrict__ flag) {
  __shared__ int32_t run_s[kWarps][64], run_p[kWarps][64];
  __shared__ int32_t site_i[kWarps][32];
  __shared__ double4 site_p[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* rs = run_s[warp];
  int32_t* rp = run_p[warp];
  int32_t* si = site_i[warp];
  double4* sp = site_p[warp];
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t c = (int64_t)blockIdx.x * kWarps + warp; c < ncell; c += nwarps) {
    const int32_t c0 = start[c], c1 = start[c + 1];
    if (c0 == c1) continue;
    const int cz = (int)(c % g.ncz), cy = (int)((c / g.ncz) % g.ncy),
              cx = (int)(c / ((int64_t)g.ncz * g.ncy));
    int xs[kSpan], ys[kSpan], zlo[2], zhi[2];
    const int nx = axis_cells(cx, g.ncx, xs), ny = axis_cells(cy, g.ncy, ys),
              nz = axis_runs(cz, g.ncz, zlo, zhi);
    const int nruns = nx * ny * nz;
    // interior cell: no candidate is across a periodic boundary and every
    // |d| < 3 cells < L/2, so wrap1(d) == d bit for bit (rint(d/L) == 0):
    // the displacement is a plain subtraction
    const bool interior = g.ncx > 3 * kSpan / 2 && g.ncy > 3 * kSpan / 2 &&
                          g.ncz > 3 * kSpan / 2 && cx >= kReach && cx + kReach < g.ncx &&
                          cy >= kReach && cy + kReach < g.ncy && cz >= kReach &&
                          cz + kReach < g.ncz;
    __syncwarp();
    int len0 = 0, len1 = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      int len = 0;
      if (r < nruns) {
        const int q = r % nz, ab = r / nz;
        const int col = (xs[ab / ny] * g.ncy + ys[ab % ny]) * g.ncz;
        const int32_t s0 = start[col + zlo[q]];
        rs[r] = s0;
        len = start[col + zhi[q] + 1] - s0;
      }
      if (h == 0) len0 = len; else len1 = len;
    }
    int inc0 = len0, inc1 = len1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(0xffffffffu, inc0, o);
      const int t1 = __shfl_up_sync(0xffffffffu, inc1, o);
      if (lane >= o) { inc0 += t0; inc1 += t1; }
    }
    const int tot0 = __shfl_sync(0xffffffffu, inc0, 31);
    rp[lane] = inc0 - len0;
    rp[lane + 32] = tot0 + inc1 - len1;
    const int total = tot0 + __shfl_sync(0xffffffffu, inc1, 31);
    auto slot_of = [&](int v) {
      int lo = 0, hi = nruns - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rp[mid] <= v) lo = mid; else hi = mid - 1;
      }
      return rs[lo] + (v - rp[lo]);
    };
    // the cell's owned sites, 32 at a time
    for (int32_t e0 = c0; e0 < c1; e0 += 32) {
      const int32_t site = (e0 + lane < c1) ? atoms[e0 + lane] : -1;
      const bool own = site >= 0 && site < n_own;
      const unsigned om = __ballot_sync(0xffffffffu, own);
      const int ns = __popc(om);
      if (ns == 0) continue;
      __syncwarp();
      if (own) {
        const int q = __popc(om & lanemask_lt());
        si[q] = site;
        sp[q] = P[site];
      }
      __syncwarp();
      int k = 0;  // row length of group site `lane`
      int32_t ja = (lane < total) ? __ldg(atoms + slot_of(lane)) : -1;
      for (int base = 0; base < total; base += 32) {
        const int vn = base + 32 + lane;
        const int32_t jb = (vn < total) ? __ldg(atoms + slot_of(vn)) : -1;
        double4 pj = make_double4(0.0, 0.0, 0.0, 0.0);
        if (ja >= 0) pj = ldg4(P + ja);
        for (int q = 0; q < ns; ++q) {
          const int32_t i = si[q];
          const double4 pi = sp[q];
          bool in = false;
          if (ja >= 0 && ja != i) {
            double dx, dy, dz;
            if (interior)
              in = dist2(__dsub_rn(pi.x, pj.x), __dsub_rn(pi.y, pj.y), __dsub_rn(pi.z, pj.z)) <= c2;
            else
              in = min_image(b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz) <= c2;
          }
          const unsigned m = __ballot_sync(0xffffffffu, in);
          const int kq = __shfl_sync(0xffffffffu, k, q);
          if (in) {
            const int32_t pos = kq + __popc(m & lanemask_lt());
            if (pos < cap) nbr[(size_t)i * (size_t)cap + pos] = ja;
          }
          if (lane == q) k += __popc(m);
        }
        ja = jb;
      }
      if (lane < ns) cnt[si[lane]] = k;
      // reference capacity rule (see k_nlist_build): rows longer than the
      // cap count their upper pairs
      unsigned big = __ballot_sync(0xffffffffu, lane < ns && k > MDG_MAX_NEIGHBORS && k <= cap);
      while (big) {
        const int q = __ffs(big) - 1;
        big &= big - 1;
        const int kq = __shfl_sync(0xffffffffu, k, q);
        const int32_t i = si[q];
        const int32_t* out = nbr + (size_t)i * (size_t)cap;
        const int32_t oi = perm[i];
        int32_t upper = 0;
        for (int e = lane; e < kq; e += 32) upper += (__ldg(perm + out[e]) > oi) ? 1 : 0;
        upper = warp_allsum_i(upper);
        if (lane == 0 && upper > MDG_MAX_NEIGHBORS) atomicMin(&flag[0], oi);
      }
    }
  }
}

// max and sum of counts -> results[slot], results[slot+1]
// max and sum of cnt[0..n) over the whole GPU in one launch: block partials
// go to integer atomics in flag[1] (max), flag[2..3] (sum, int64) and the
// last block to finish publishes them and resets the scratch (integer
// arithmetic, so the result is order-independent).
__global__ void k_count_stats(int64_t n, const int32_t* __restrict__ cnt,
                              double* __restrict__ results, int slot, int32_t* __restrict__ flag) {
  __shared__ long long s_sum[8];
  __shared__ int s_max[8];
  __shared__ bool last;
  long long sum = 0;
  int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = cnt[i];
    sum += v;
    mx = max(mx, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { s_sum[warp] = sum; s_max[warp] = mx; }
  __syncthreads();
  unsigned long long* gsum = reinterpret_cast<unsigned long long*>(flag + 2);
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { sum += s_sum[w]; mx = max(mx, s_max[w]); }
    atomicMax(flag + 1, mx);
    atomicAdd(gsum, (unsigned long long)sum);
    __threadfence();
    last = (atomicAdd(flag + 4, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    results[slot] = (double)*(volatile int*)(flag + 1);
    results[slot + 1] = (double)(long long)*(volatile unsigned long long*)gsum;
    flag[1] = 0;
    *gsum = 0ull;
    flag[4] = 0;
  }
}

void count_stats_n(mdg_ctx* c, const int32_t* cnt, int64_t n, int slot) {
  const unsigned blocks = (unsigned)std::min<int64_t>(296, std::max<int64_t>(1, grid_for(n, 256)));
  MDG_LAUNCH(c, "count_stats", blocks, 256, 0, k_count_stats, n, cnt, c->results, slot,
             c->d_flag);
}

void count_stats(mdg_ctx* c, const int32_t* cnt, int slot) { count_stats_n(c, cnt, c->n_own, slot); }

// Sort every row ascending by j: with Morton-ordered sites, consecutive j of
// a sorted row share cache lines, so the pair kernels' 32-lane gathers touch
// fewer lines. Bitonic network over the warp: element e = r * 32 + lane lives
// in register r of `lane`; strides < 32 exchange by shuffle, larger ones
// within the lane. R = padded row length / 32 (a power of two).
template <int R>
__device__ __forceinline__ void sort_row(int32_t* __restrict__ row, int m, int lane) {
  int32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = r * 32 + lane;
    v[r] = (e < m) ? row[e] : 0x7fffffff;
  }
#pragma unroll
  for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if ((r & jr) == 0) {
            const int e = r * 32 + lane;
            const bool asc = (e & k) == 0;
            const int32_t a = v[r], b = v[r | jr];
            if ((a > b) == asc) { v[r] = b; v[r | jr] = a; }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = r * 32 + lane;
          const int32_t b = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool keep_min = ((e & j) == 0) == ((e & k) == 0);
          v[r] = keep_min ? min(v[r], b) : max(v[r], b);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = r * 32 + lane;
    if (e < m) row[e] = v[r];
  }
}

// One launch sorts every row of up to 32 RMAX slots, each padded only to the
// next power of two of its own length (a 9.5 A row of ~330 slots sorts as 512,
// not as the list's longest row). flag (may be NULL): sort only when *flag
// (the device-decided cut of kernel_rows).
template <int RMAX>
__global__ void __launch_bounds__(kBlock) k_sort_rows(int64_t n, int32_t* __restrict__ nbr,
                                                    const int32_t* __restrict__ cnt, int32_t cap,
                                                    const int32_t* __restrict__ flag, int lo) {
  if (flag && *flag == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kBlock / 32);
  for (int64_t i = blockIdx.x * (int64_t)(kBlock / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const int m = cnt[i];
    if (m < 2 || m <= lo || m > 32 * RMAX) continue;
    int32_t* row = nbr + (size_t)i * cap;
    if (m <= 32) sort_row<1>(row, m, lane);
    else if (RMAX >= 2 && m <= 64) sort_row<(RMAX >= 2 ? 2 : 1)>(row, m, lane);
    else if (RMAX >= 4 && m <= 128) sort_row<(RMAX >= 4 ? 4 : 1)>(row, m, lane);
    else if (RMAX >= 8 && m <= 256) sort_row<(RMAX >= 8 ? 8 : 1)>(row, m, lane);
    else if (RMAX >= 16 && m <= 512) sort_row<(RMAX >= 16 ? 16 : 1)>(row, m, lane);
    else if (RMAX >= 32) sort_row<(RMAX >= 32 ? 32 : 1)>(row, m, lane);
  }
}

// Sort the rows (<= 1024 slots) of nbr/cnt in one launch sized by max_cnt.
// Returns false when sorting is disabled (MDG_SORT_ROWS=0).
static bool sort_rows(mdg_ctx* c, int32_t* nbr, const int32_t* cnt, int32_t cap,
                      int32_t max_cnt, const int32_t* flag = nullptr) {
  static const int enabled = [] {
    const char* e = getenv("MDG_SORT_ROWS");
    return e ? atoi(e) : 1;
  }();
  // sorted rows also let the half-row kernels start at the first j > i
  // (row_suffix; rows longer than 1024 stay unsorted and are walked whole)
  if (!enabled) return false;
  if (max_cnt < 2) return true;
  const int64_t rows = c->n_own;
  const unsigned grid = (unsigned)std::min<int64_t>(148 * 16, (rows + 3) / 4);
  const int need = (std::min(1024, (int)max_cnt) + 31) / 32;
  // rows up to 512 slots in a 16-register-row launch; only the longer ones
  // pay the 32-register variant's occupancy
#define MDG_SORT(R, LO) \
  MDG_LAUNCH(c, "sort_rows", grid, kBlock, 0, k_sort_rows<R>, rows, nbr, cnt, cap, flag, LO)
  if (need <= 1) MDG_SORT(1, 0);
  else if (need <= 2) MDG_SORT(2, 0);
  else if (need <= 4) MDG_SORT(4, 0);
  else if (need <= 8) MDG_SORT(8, 0);
  else if (need <= 16) MDG_SORT(16, 0);
  else {
    MDG_SORT(16, 0);
    MDG_SORT(32, 512);
  }
#undef MDG_SORT
  return true;
}

static void ensure_list_storage(mdg_ctx* c, DevList& L, int32_t cap) {
  const size_t need = (size_t)c->n_own * (size_t)cap;
  if (need > L.nbr_elems) {
    if (L.nbr) cudaFree(L.nbr);
    L.nbr = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&L.nbr, need * sizeof(int32_t)));
    L.nbr_elems = need;
  }
  if (!L.cnt) MDG_CUDA_CHECK(cudaMalloc(&L.cnt, (size_t)c->n_cap * sizeof(int32_t)));
  L.cap = cap;
}

void nlist_build(mdg_ctx* c, int list_id, double list_cutoff, int sites) {
  DevList& L = c->lists[list_id];
  const double4* P = (sites == MDG_SITES_VDW) ? c->vsite : c->pos;
  Grid g;
  // edge >= list_cutoff / kReach: the (2 kReach + 1)^3 stencil covers a
  // sphere-sized region with ~40% fewer candidates than 27 full-size cells
  const double cell_min = list_cutoff / kReach;
  g.ncx = std::max(1, (int)(c->lx / cell_min));
  g.ncy = std::max(1, (int)(c->ly / cell_min));
  g.ncz = std::max(1, (int)(c->lz / cell_min));
  g.ex = c->lx / g.ncx;
  g.ey = c->ly / g.ncy;
  g.ez = c->lz / g.ncz;
  const int64_t ncell = (int64_t)g.ncx * g.ncy * g.ncz;
  if (ncell + 1 > c->cell_cap) {
    if (c->cell_start) cudaFree(c->cell_start);
    if (c->cell_fill) cudaFree(c->cell_fill);
    c->cell_start = c->cell_fill = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&c->cell_start, (ncell + 1) * sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMalloc(&c->cell_fill, (ncell + 1) * sizeof(int32_t)));
    c->cell_cap = ncell + 1;
  }
  const int64_t n = c->n;
  MDG_CUDA_CHECK(cudaMemsetAsync(c->cell_fill, 0, ncell * sizeof(int32_t), c->stream));
  MDG_LAUNCH(c, "cell_assign", grid_for(n, 256), 256, 0, k_cell_assign, n, P, g, c->cell_of,
             c->cell_fill);
  // k_scan reads counts from cell_fill and rewrites it as the fill cursor
  MDG_LAUNCH(c, "cell_scan", 1, 1024, 0, k_scan, ncell, c->cell_fill, c->cell_start,
             c->cell_fill);
  MDG_LAUNCH(c, "cell_fill", grid_for(n, 256), 256, 0, k_cell_fill, n, c->cell_of, c->cell_fill,
             c->cell_atoms);
  MDG_LAUNCH(c, "cell_sort", grid_for(ncell, 128), 128, 0, k_cell_sort, ncell, c->cell_start,
             c->cell_atoms);

  // capacity: density estimate, grown to the measured maximum if exceeded
  const double vol = c->lx * c->ly * c->lz;
  const double expect = (double)c->n_global / vol * 4.18879020478639 * list_cutoff * list_cutoff *
                        list_cutoff;
  int32_t cap = (int32_t)std::min<double>((double)c->max_pairs, 1.35 * expect + 48.0);
  cap = std::max<int32_t>(32, (cap + 31) & ~31);
  if (L.cap > cap && L.nbr) cap = L.cap;
  const Box b = make_box(c->lx, c->ly, c->lz);
  const double c2 = list_cutoff * list_cutoff;
  const int64_t rows = c->n_own;  // rows for owned sites; candidates span the halo too
  const int64_t ipb = sites_per_block((const void*)k_nlist_build, rows);
  const unsigned ngrid = (unsigned)((rows + ipb - 1) / ipb);
  // cell-per-warp kernel (MDG_CELL_BUILD=0: the per-site kernel)
  static const int cell_build = env_int("MDG_CELL_BUILD", 1);
  const bool use_cells = cell_build != 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    ensure_list_storage(c, L, cap);
    MDG_CUDA_CHECK(cudaMemsetAsync(c->d_flag, 0x7f, sizeof(int32_t), c->stream));
    if (use_cells) {
      MDG_LAUNCH(c, "nlist_cells", (unsigned)std::min<int64_t>((ncell + kWarps - 1) / kWarps, 148 * 64),
                 kBlock, 0, k_nlist_cells, ncell, rows, P, g, c->cell_start, c->cell_atoms, b, c2,
                 cap, L.nbr, L.cnt, c->d_perm, c->d_flag);
    } else {
      MDG_LAUNCH(c, "nlist_build", ngrid, kBlock, 0, k_nlist_build, rows, (int)ipb, P,
                 c->cell_of, g, c->cell_start, c->cell_atoms, b, c2, cap, L.nbr, L.cnt,
                 c->d_perm, c->d_flag);
    }
    count_stats(c, L.cnt, 60);
    int32_t bad_site = 0;
    MDG_CUDA_CHECK(cudaMemcpyAsync(&bad_site, c->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                   c->stream));
    fetch_results(c);
    if (bad_site != 0x7f7f7f7f) {
      L.valid = false;
      throw_error(MDG_CAPACITY, "neighbor table: site " + std::to_string(bad_site) +
                                    " exceeds the per-site neighbor capacity");
    }
    const int32_t mx = (int32_t)c->h_results[60];
    const int64_t sum = (int64_t)c->h_results[61];
    if (mx > c->max_pairs) {
      L.valid = false;
      throw_error(MDG_CAPACITY, "neighbor table: a site exceeds the per-site neighbor capacity (" +
                                    std::to_string(mx) + " > " + std::to_string(c->max_pairs) +
                                    ")");
    }
    if (mx <= cap) {
      // rows stay in candidate order here; kernel_rows sorts the rows the
      // kernels walk (the buffered cut, or this list on its first use)
      L.sorted = false;
      L.valid = true;
      L.version = ++c->epoch;
      L.cutoff = list_cutoff;
      L.sites = sites;
      L.max_cnt = mx;
      L.half_pairs = sum / 2;
      list_snapshot(c, list_id);
      debug_check_rows(c, "list", L.nbr, L.cnt, L.cap, rows, c->n, false);
      return;
    }
    cap = (mx + 31) & ~31;
  }
  throw_error(MDG_CUDA, "nlist_build: capacity retry failed");
}

// ---- buffered inner lists (dynamic pruning) ---------------------------------
// flag = 1 when some site has moved more than half the buffer since the cut
// (minimum image: a site wrapped back into the box across a face has moved
// only its step's distance)
__global__ void k_moved(int64_t n, Box b, const double4* __restrict__ P,
                        const double4* __restrict__ ref, double lim2,
                        int32_t* __restrict__ flag) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool moved = false;
  if (s < n) {
    const double4 p = P[s], r = ref[s];
    double dx, dy, dz;
    moved = min_image(b, p.x, p.y, p.z, r.x, r.y, r.z, dx, dy, dz) > lim2;
  }
  if (__any_sync(0xffffffffu, moved) && (threadIdx.x & 31) == 0) *flag = 1;
}

struct CutArgs {
  int64_t n_rows, n_all;
  int ipw;
  const double4* __restrict__ P;
  ListView src;
  Box b;
  double rc2;
  int32_t* __restrict__ nbr;
  int32_t* __restrict__ cnt;
  double4* __restrict__ ref;
  const int32_t* __restrict__ flag;
  int32_t* __restrict__ cuts;  // mapped host counter
  int32_t* __restrict__ gen;   // device cut generation
  double* __restrict__ partials;  // unused (launch macro contract)
  // list staleness: sites' positions when the source list was built, the
  // largest motion the cut can tolerate (squared), the sticky result slot
  const double4* __restrict__ ref0;
  double lim0_2, warn0_2;
  double* __restrict__ stale;
  int32_t* __restrict__ warn;
  int32_t gen0;  // list generation the warning refers to
};

// When *flag: every owned row keeps its slots with r^2 <= rc^2 (the
// reference's wrap1/dist2 test, order kept: sorted rows stay sorted) and the
// reference positions are refreshed for all sites. Otherwise returns at once.
__global__ void __launch_bounds__(kBlock) k_cut_rows(CutArgs a) {
  if (*a.flag == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid == 0 && *a.flag == 1) atomicAdd_system(a.cuts, 1);  // motion cuts only (2: forced)
  if (tid == 0) atomicAdd(a.gen, 1);  // every cut: the rows' generation
  for (int64_t s = tid; s < a.n_all; s += (int64_t)gridDim.x * blockDim.x) a.ref[s] = a.P[s];
  MDG_SITE_LOOP(i, a.n_rows, a.ipw) {
    const double4 pi = a.P[i];
    if (lane == 0 && a.ref0) {  // the source list misses pairs once a site moved too far
      const double4 r0 = a.ref0[i];
      double dx, dy, dz;
      const double d2 = min_image(a.b, pi.x, pi.y, pi.z, r0.x, r0.y, r0.z, dx, dy, dz);
      if (d2 > a.lim0_2) *a.stale = 1.0;
      if (d2 > a.warn0_2 && a.warn) *a.warn = a.gen0;
    }
    const int c = a.src.cnt[i];
    const int32_t* row = list_row(a.src, i);
    int32_t* out = a.nbr + (size_t)i * a.src.cap;
    int kept = 0;
    for (int base = 0; base < c; base += 32) {
      const int k = base + lane;
      const int32_t j = k < c ? __ldg(row + k) : 0;
      bool keep = false;
      if (k < c) {
        const double4 pj = ldg4(a.P + (j & 0x7fffffff));
        double dx, dy, dz;
        keep = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz) <= a.rc2;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) out[kept + __popc(m & lanemask_lt())] = j;
      kept += __popc(m);
    }
    if (lane == 0) a.cnt[i] = kept;
  }
}

// A kernel walking list rows with cutoff rc sees every pair within rc only
// while no site has moved more than (list cutoff - rc) / 2 since the list
// was built: past that, result slot kStaleSlot + list id turns 1 (sticky
// until the list is rebuilt; the host raises MDG_CONTRACT at its next read
// of the results, check_lists_fresh).
__global__ void k_list_motion(int64_t n, Box b, const double4* __restrict__ P,
                              const double4* __restrict__ ref0, double lim2, double warn2,
                              double* __restrict__ stale, int32_t* __restrict__ warn,
                              int32_t gen) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (s < n) {
    const double4 p = P[s], r = ref0[s];
    double dx, dy, dz;
    d2 = min_image(b, p.x, p.y, p.z, r.x, r.y, r.z, dx, dy, dz);
  }
  if (__any_sync(0xffffffffu, d2 > lim2) && (threadIdx.x & 31) == 0) *stale = 1.0;
  if (__any_sync(0xffffffffu, d2 > warn2) && (threadIdx.x & 31) == 0 && warn) *warn = gen;
}

// positions at the build of list_id (the staleness reference)
void list_snapshot(mdg_ctx* c, int list_id) {
  DevList& L = c->lists[list_id];
  if (!L.ref0) MDG_CUDA_CHECK(cudaMalloc(&L.ref0, (size_t)c->n_cap * sizeof(double4)));
  const double4* P = (L.sites == MDG_SITES_VDW) ? c->vsite : c->pos;
  MDG_CUDA_CHECK(cudaMemcpyAsync(L.ref0, P, (size_t)c->n * sizeof(double4),
                                 cudaMemcpyDeviceToDevice, c->stream));
  MDG_CUDA_CHECK(cudaMemsetAsync(c->results + kStaleSlot + list_id, 0, sizeof(double), c->stream));
  ++c->list_gen;
}

void check_lists_fresh(const mdg_ctx* c) {
  for (int l = 0; l < MDG_MAX_LISTS; ++l)
    if (c->h_results[kStaleSlot + l] != 0.0)
      throw_error(MDG_CONTRACT, "neighbour list " + std::to_string(l) +
                                    " outdated: sites moved more than half its skin since it was "
                                    "built (rebuild it more often)");
}

ListView kernel_rows(mdg_ctx* c, int list_id, double rc, bool want_sorted) {
  DevList& L = c->lists[list_id];
  auto full_rows = [&] {
    if (!L.sorted) L.sorted = sort_rows(c, L.nbr, L.cnt, L.cap, L.max_cnt);
    if (L.ref0 && L.cutoff > rc) {
      const double lim = 0.5 * (L.cutoff - rc);
      const double4* P = (L.sites == MDG_SITES_VDW) ? c->vsite : c->pos;
      MDG_LAUNCH(c, "list_motion", grid_for(c->n, 256), 256, 0, k_list_motion, c->n,
                 make_box(c->lx, c->ly, c->lz), P, (const double4*)L.ref0, lim * lim,
                 0.36 * lim * lim, c->results + kStaleSlot + list_id, c->d_warn, c->list_gen);
    }
    return ListView{L.nbr, L.cnt, L.cap, L.sorted};
  };
  const ListView full{L.nbr, L.cnt, L.cap, false};  // cut source: any order
  // buffer (A): MDG_PRUNE_BUFFER, 0 = walk the full list
  // (read per call: tests switch it)
  const char* eb = std::getenv("MDG_PRUNE_BUFFER");
  const double buf = eb ? std::atof(eb) : 0.5;
  // small systems: the per-call check and gated launches cost more than the
  // shorter rows save (MDG_PRUNE_MIN_SITES)
  const int min_sites = env_int("MDG_PRUNE_MIN_SITES", 50000);
  const double rcut = rc + buf;
  if (buf <= 0 || rcut >= L.cutoff || c->n_own < min_sites) return full_rows();
  DevList::Inner& I = L.inner;
  if (!I.hcuts) {
    MDG_CUDA_CHECK(cudaHostAlloc(&I.hcuts, sizeof(int32_t), cudaHostAllocMapped));
    *I.hcuts = 0;
    MDG_CUDA_CHECK(cudaHostGetDevicePointer(&I.dcuts, I.hcuts, 0));
  }
  if (I.bypass > 0) {
    --I.bypass;
    return full_rows();
  }
  if (++I.calls >= 2) {  // motion cuts on both of the last 2 calls: bypass the next 128
    const int cuts = *(volatile int32_t*)I.hcuts;
    if (cuts - I.cuts0 >= I.calls) {
      I.bypass = 128;
      I.src_version = -1;  // cut afresh afterwards
    }
    I.calls = 0;
    I.cuts0 = cuts;
    if (I.bypass) return full_rows();
  }
  const size_t need = (size_t)c->n_own * (size_t)L.cap;
  if (need > I.elems) {
    if (I.nbr) cudaFree(I.nbr);
    I.nbr = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&I.nbr, need * sizeof(int32_t)));
    I.elems = need;
    I.src_version = -1;
  }
  if (!I.cnt) MDG_CUDA_CHECK(cudaMalloc(&I.cnt, (size_t)c->n_cap * sizeof(int32_t)));
  if (!I.ref) MDG_CUDA_CHECK(cudaMalloc(&I.ref, (size_t)c->n_cap * sizeof(double4)));
  if (!I.flag) MDG_CUDA_CHECK(cudaMalloc(&I.flag, sizeof(int32_t)));
  if (!I.gen) {
    MDG_CUDA_CHECK(cudaMalloc(&I.gen, sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMemsetAsync(I.gen, 0, sizeof(int32_t), c->stream));
  }
  const double4* P = (L.sites == MDG_SITES_VDW) ? c->vsite : c->pos;
  // rows cut without a sort do not serve a caller that needs them sorted
  const bool stale =
      I.src_version != L.version || I.rc != rcut || (want_sorted && !I.cut_sorted);
  if (stale) {
    // cut unconditionally (2: forced, not counted as motion by the bypass)
    MDG_CUDA_CHECK(cudaMemsetAsync(I.flag, 0, sizeof(int32_t), c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(I.flag, 2, 1, c->stream));
    I.src_version = L.version;
    I.rc = rcut;
  } else {
    MDG_CUDA_CHECK(cudaMemsetAsync(I.flag, 0, sizeof(int32_t), c->stream));
    const double half = 0.5 * buf;
    MDG_LAUNCH(c, "moved", grid_for(c->n, 256), 256, 0, k_moved, c->n,
               make_box(c->lx, c->ly, c->lz), P, I.ref, half * half, I.flag);
  }
  CutArgs k;
  k.n_rows = c->n_own;
  k.n_all = c->n;
  k.P = P;
  k.src = full;
  k.b = make_box(c->lx, c->ly, c->lz);
  k.rc2 = rcut * rcut;
  k.nbr = I.nbr;
  k.cnt = I.cnt;
  k.ref = I.ref;
  k.flag = I.flag;
  k.cuts = I.dcuts;
  k.gen = I.gen;
  k.ref0 = L.ref0;
  k.lim0_2 = 0.25 * (L.cutoff - rcut) * (L.cutoff - rcut);
  k.warn0_2 = 0.36 * k.lim0_2;  // 0.6 x the tolerable motion
  k.stale = c->results + kStaleSlot + list_id;
  k.warn = c->d_warn;
  k.gen0 = c->list_gen;
  MDG_LAUNCH_SITES(c, "cut_rows", k.n_rows, k, k_cut_rows);
  // the cut rows are short: sort them (bucketed by length), when cut -- unless
  // the caller walks them in any order (then a later cut for a caller that
  // needs them sorted is forced, above)
  if (stale) I.cut_sorted = want_sorted;
  const bool sorted = I.cut_sorted && sort_rows(c, I.nbr, I.cnt, L.cap, L.max_cnt, I.flag);
  debug_check_rows(c, "inner", I.nbr, I.cnt, L.cap, c->n_own, c->n, sorted);
  return ListView{I.nbr, I.cnt, L.cap, sorted, true};
}

}  // namespace mdg
