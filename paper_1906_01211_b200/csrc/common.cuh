// common.cuh -- device helpers shared by every pair kernel.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "mdg_internal.h"

// Debug build (make debug: -DMDG_DEBUG, libmdg_debug.so): device asserts on
// list / ring / slot bounds, and a full check of every list the kernels walk
// (debug.cu). The substitute for compute-sanitizer, which is closed on this
// pool. Compiled out of the product build.
#ifdef MDG_DEBUG
#include <cassert>
#define MDG_DASSERT(c) assert(c)
#else
#define MDG_DASSERT(c) ((void)0)
#endif

namespace mdg {

// proj/include/mdvec/pbc.hpp:27-31, op for op: DMUL, FRND (round-half-even
// = nearbyint), DFMA, DSETP, DADD. The explicit _rn intrinsics forbid
// contraction so pair membership is bit-identical to the reference.
__device__ __forceinline__ double wrap1(double d, double L, double invL, double halfL) {
  const double t = __fma_rn(-rint(__dmul_rn(d, invL)), L, d);
  return (t >= halfL) ? __dsub_rn(t, L) : t;
}

// proj/include/mdvec/pbc.hpp:35-37
__device__ __forceinline__ double dist2(double dx, double dy, double dz) {
  return __fma_rn(dx, dx, __fma_rn(dy, dy, __dmul_rn(dz, dz)));
}

// The w word of pos / vsite carries the site's exclusion group (an integer
// value as a double), so the pair prologues test exclusions on the gathered
// position instead of a second gather (Halgren 3.11 -> 2.96 ms). (The
// permanent-field pass keeps its int32 group gather: measured faster there.)
// Bit layout of w: low word = exclusion group, high word = vdW parameter type
// (mdg_ctx::vtab). Only moved and compared as integers, never used in FP math.
__device__ __forceinline__ double group_bits(int32_t g, int32_t type) {
  return __hiloint2double(type, g);
}

__device__ __forceinline__ bool same_group(const double4& a, const double4& b) {
  return __double2loint(a.w) == __double2loint(b.w);
}

// d = r_i - r_j, minimum image; returns r2
__device__ __forceinline__ double min_image(const Box& b, double xi, double yi, double zi,
                                            double xj, double yj, double zj, double& dx,
                                            double& dy, double& dz) {
  dx = wrap1(__dsub_rn(xi, xj), b.lx, b.ix, b.hx);
  dy = wrap1(__dsub_rn(yi, yj), b.ly, b.iy, b.hy);
  dz = wrap1(__dsub_rn(zi, zj), b.lz, b.iz, b.hz);
  return dist2(dx, dy, dz);
}

// ---- bulk asynchronous copies (TMA engine) into shared memory, completion
// tracked by mbarrier transaction counts
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}


// One 256-bit read-only load per lane (sm_100a LDG.E.ENL2.256): a gathered
// 32-B record costs one L1 wavefront per distinct sector instead of two
// LDG.128 instructions. All double4 arrays are 32-B aligned.
__device__ __forceinline__ double4 ldg4(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of NV values into partials[blockIdx.x][*].
// Block size must be kBlock (4 warps).
template <int NV>
__device__ __forceinline__ void block_store_partials(double (&v)[NV], double* partials) {
  __shared__ double red[kBlock / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) red[warp][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kBlock / 32; ++w) s += red[w][threadIdx.x];
    partials[(size_t)blockIdx.x * kRedVals + threadIdx.x] = s;
  }
}

// Thole factors (proj/include/mdvec/polar.hpp:55-62) with per-site
// pdamp = alpha^(1/6): u = r/(pd_i pd_j), formed by the callers as
// r * ipd_i * ipd_j from the stored inverses (no division). l7 for the
// quadrupole field.
__device__ __forceinline__ void thole3(double u, double a, double& l3, double& l5) {
  const double au3 = a * u * u * u;
  const double ex = exp(-au3);
  l3 = 1.0 - ex;
  l5 = 1.0 - (1.0 + au3) * ex;
}

__device__ __forceinline__ void thole7(double u, double a, double& l3, double& l5,
                                       double& l7) {
  const double au3 = a * u * u * u;
  const double ex = exp(-au3);
  l3 = 1.0 - ex;
  l5 = 1.0 - (1.0 + au3) * ex;
  l7 = 1.0 - (1.0 + au3 + 0.6 * au3 * au3) * ex;
}

// erfc(x) from the exp(-x^2) the Ewald recursion computes anyway:
// erfc = exp(-x^2) * erfcx(x), erfcx on [0, 6] a degree-18 polynomial in
// t = (x - 3)/(x + 3) (tools/fit_erfcx.py: max relative error 4.4e-16 in
// double Horner). Coefficients sit in the constant bank, so the DFMAs take
// them as operands (the library erfc materialises its constants with UMOVs
// and recomputes exp(-x^2) internally). Beyond x = 6 (erfc < 2e-17) or for
// NaN the library function is used.
static __constant__ double kErfcx[19] = {
    0.17900115118138996,     -0.32623356004303744,    0.24560380171233284,
    -0.15011593650073177,    0.07166583719787115,     -0.024392499321270803,
    0.004269136332174619,    0.0007077465012785561,   -0.0005970618259925815,
    4.525468578951527e-05,   6.405418474854186e-05,   -1.285998407416855e-05,
    -7.962426888254932e-06,  2.146772173006056e-06,   1.2424066961151949e-06,
    -3.9301447303001125e-07, -3.9867716616971016e-07, -1.1020487050346528e-07,
    -1.1194382877771014e-08};

__device__ __forceinline__ double rcp_nr(double d) {
  float f;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"((float)d));
  double y = (double)f;  // ~1e-7, two Newton steps -> full double precision
  double e = __fma_rn(-d, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-d, y, 1.0);
  return __fma_rn(y, e, y);
}

__device__ __forceinline__ double erfc_from_exp(double x, double exp_mx2) {
  if (!(x <= 6.0)) return erfc(x);
  const double t = (x - 3.0) * rcp_nr(x + 3.0);
  double p = kErfcx[18];
#pragma unroll
  for (int k = 17; k >= 0; --k) p = __fma_rn(p, t, kErfcx[k]);
  return exp_mx2 * p;
}

// Tinker bn recursion for real-space Ewald: B0 = erfc(ar)/r,
// Bn = ((2n-1) B(n-1) + (2a^2)^n/(a sqrt(pi)) exp(-a^2 r^2)) / r^2.
// Callers pass 1/r (their one division per pair) and 1/r^2 = (1/r)^2.
template <int NMAX>
__device__ __forceinline__ void ewald_bn(double r, double inv_r, double inv_r2, double alpha,
                                         double (&bn)[NMAX + 1]) {
  const double ralpha = alpha * r;
  const double alsq2 = 2.0 * alpha * alpha;
  // (2a^2)^n / (a sqrt(pi)) = (2a / sqrt(pi)) (2a^2)^(n-1): no division
  // (the compiler does not hoist a per-pair 1 / (a sqrt(pi)) out of the row)
  double alsq2n = 1.1283791670955125739 * alpha;
  const double exp2a = exp(-ralpha * ralpha);
  bn[0] = erfc_from_exp(ralpha, exp2a) * inv_r;
#pragma unroll
  for (int k = 1; k <= NMAX; ++k) {
    if (k > 1) alsq2n *= alsq2;
    bn[k] = ((double)(2 * k - 1) * bn[k - 1] + alsq2n * exp2a) * inv_r2;
  }
}

// Neighbour lists are row-major: site i's row starts at nbr + i * cap (cap a
// multiple of 32, so every row is 128-B aligned) and holds cnt[i] entries.
struct ListView {
  const int32_t* nbr;
  const int32_t* cnt;
  int32_t cap;
  bool sorted = false;  // rows ascending in (j & 0x7fffffff)
  bool dense = false;   // buffered cut rows: nearly every slot in range (DIRECT walk)
};

// Rows a kernel with cutoff rc walks over list `list_id`: the buffered inner
// list (rows cut to rc + buffer, re-cut on the device when some site has moved
// more than buffer/2 since the last cut) or the list itself (nlist.cu).
// want_sorted false: the caller walks the rows in any order (the cluster
// kernels' hash-built unions), so a cut skips the row sort.
ListView kernel_rows(mdg_ctx* c, int list_id, double rc, bool want_sorted = true);

__device__ __forceinline__ const int32_t* list_row(const ListView& L, int64_t i) {
  return L.nbr + (size_t)i * (size_t)L.cap;
}

// First slot of a sorted row whose neighbour (flag bit masked) is > i: the
// half-row kernels walk only that suffix. Two dependent probes: 32 evenly
// spaced slots, then the <= 31 slots between the bracketing probes. Rows
// longer than 1024 return 0 (the kernels' prologue still drops j < i).
__device__ __forceinline__ int row_suffix(const int32_t* __restrict__ row, int cnt, int64_t i,
                                          int lane) {
  if (cnt == 0 || cnt > 1024) return 0;
  const int step = (cnt + 31) >> 5;
  const int nvalid = (cnt + step - 1) / step;
  const bool v = lane < nvalid;
  const bool gt = v && (int64_t)(__ldg(row + lane * step) & 0x7fffffff) > i;
  const unsigned m = __ballot_sync(0xffffffffu, gt);
  int lo, hi;
  if (m == 0) {
    lo = (nvalid - 1) * step + 1;
    hi = cnt;
  } else {
    const int p = __ffs(m) - 1;
    if (p == 0) return 0;
    lo = (p - 1) * step + 1;
    hi = p * step;
  }
  const bool gt2 = (lo + lane < hi) && (int64_t)(__ldg(row + lo + lane) & 0x7fffffff) > i;
  const unsigned m2 = __ballot_sync(0xffffffffu, gt2);
  return m2 ? lo + __ffs(m2) - 1 : hi;
}

// Minimum resident blocks per SM of the warp-per-site pair kernels (register
// caps); tuned per kernel on config 4, overridable for experiments.
// (An explicit minimum of 1 lifts nvcc's default register heuristic and
// costs occupancy: multipoles 5.04 ms at 204 registers vs 4.4 at <= 170.)
#ifndef MDG_MPOLE_MINB
#define MDG_MPOLE_MINB 3
#endif
#ifndef MDG_HALGREN_MINB
#define MDG_HALGREN_MINB 5
#endif
#ifndef MDG_POLFORCE_MINB
#define MDG_POLFORCE_MINB 3
#endif

// ---- warp-per-site execution ------------------------------------------------
// One warp walks one site's row 32 slots at a time (coalesced 128-B index
// loads), evaluates the cheap prologue (minimum image, cutoff, exclusion) on
// every slot, and compacts the in-range pairs with a ballot into a per-warp
// shared-memory ring. The expensive pair body then always runs on 32 live
// lanes; only the final drain of a row is partial. Each warp owns `ipw`
// consecutive (spatially adjacent) sites, so a block's rows share cache lines.
constexpr int kWarps = kBlock / 32;
constexpr int kRing = 64;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_allsum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Ring {
  double4* q;  // kRing entries: (dx, dy, dz, j as bits)
  int head;    // warp-uniform
  int count;   // warp-uniform
};

// entry w: low word = j (with any flag bit), high word = j's vdW type
__device__ __forceinline__ void ring_push(Ring& r, bool in, double dx, double dy, double dz,
                                          int32_t j, int32_t type) {
  const unsigned m = __ballot_sync(0xffffffffu, in);
  MDG_DASSERT(r.count >= 0 && r.count + __popc(m) <= kRing);
  if (in) {
    const int pos = (r.head + r.count + __popc(m & lanemask_lt())) & (kRing - 1);
    r.q[pos] = make_double4(dx, dy, dz, __hiloint2double(type, j));
  }
  r.count += __popc(m);
  __syncwarp();
}

// Take `take` (<= 32) entries; lane l gets entry l when l < take.
__device__ __forceinline__ double4 ring_take(Ring& r, int take, int lane) {
  MDG_DASSERT(take >= 0 && take <= 32 && take <= r.count);
  double4 e = make_double4(0, 0, 0, 0);
  if (lane < take) e = r.q[(r.head + lane) & (kRing - 1)];
  r.head = (r.head + take) & (kRing - 1);
  r.count -= take;
  __syncwarp();
  return e;
}

__device__ __forceinline__ int32_t ring_j(const double4& e) { return __double2loint(e.w); }

__device__ __forceinline__ int32_t ring_type(const double4& e) { return __double2hiint(e.w); }

// Walk one site's row with the warp: software-pipelined so the index load of
// chunk c+2 and the position gather of chunk c+1 are in flight while chunk c
// is tested and compacted and the body runs (the kernels are latency-bound
// otherwise). pro(raw, pj, dx, dy, dz) -> in-range?; body(entry, slot) runs
// on compacted entries, slot = running index of the entry in the row's
// in-range sequence (for kernels that write a pruned row). Returns the number
// of in-range entries.
// `mol` (may be NULL) is gathered with the positions so the exclusion test
// does not wait on its own load; pro(raw, pj, mol_j, dx, dy, dz).
// TYPED: the ring entries also carry j's site type (high word of pj.w) for
// bodies that read per-type tables (ring_type); off, the entry is (dx, dy,
// dz, j) only -- the extra live word cost the register-capped field pass.
// DIRECT: no compaction -- the in-range lanes run the body on their own slot.
// For rows that are nearly all in range (the 7 A pruned rows, the buffered
// cut rows: ~85 %) the ring's shared-memory round trip (32 B in, 32 B out per
// pair, on the same L1 data pipe as the gathers) costs more than the idle
// lanes; for full skin rows (~50 % in range) the ring wins.
template <bool TYPED = false, bool DIRECT = false, class Pro, class Body>
__device__ __forceinline__ int run_row(const int32_t* __restrict__ row, int cnt, int lane,
                                       const double4* __restrict__ P,
                                       const int32_t* __restrict__ mol, Ring& ring, Pro&& pro,
                                       Body&& body) {
  MDG_DASSERT(cnt >= 0);
  int32_t ja = (lane < cnt) ? __ldg(row + lane) : 0;
  double4 pa = ldg4(P + (ja & 0x7fffffff));
  int32_t ma = mol ? __ldg(mol + (ja & 0x7fffffff)) : 0;
  int32_t jb = (32 + lane < cnt) ? __ldg(row + 32 + lane) : 0;
  int taken = 0;
  for (int base = 0; base < cnt; base += 32) {
    double4 pb = make_double4(0, 0, 0, 0);
    int32_t jc = 0, mb = 0;
    if (base + 32 < cnt) {
      pb = ldg4(P + (jb & 0x7fffffff));
      if (mol) mb = __ldg(mol + (jb & 0x7fffffff));
    }
    if (base + 64 + lane < cnt) jc = __ldg(row + base + 64 + lane);
    double dx = 0, dy = 0, dz = 0;
    const bool in = (base + lane < cnt) && pro(ja, pa, ma, dx, dy, dz);
    if constexpr (DIRECT) {
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (in)
        body(make_double4(dx, dy, dz, __hiloint2double(TYPED ? __double2hiint(pa.w) : 0, ja)),
             taken + __popc(m & lanemask_lt()));
      taken += __popc(m);
    } else {
      ring_push(ring, in, dx, dy, dz, ja, TYPED ? __double2hiint(pa.w) : 0);
      if (ring.count >= 32) {
        body(ring_take(ring, 32, lane), taken + lane);
        taken += 32;
      }
    }
    ja = jb;
    pa = pb;
    ma = mb;
    jb = jc;
  }
  if (ring.count > 0) {
    const int take = ring.count;
    const double4 e = ring_take(ring, take, lane);
    if (lane < take) body(e, taken + lane);
    taken += take;
  }
  return taken;
}

// Site loop of a warp-per-site kernel launched by MDG_LAUNCH_SITES: block b
// owns sites [b*ipb, (b+1)*ipb), its warps take every kWarps-th site.
#define MDG_SITE_LOOP(i, n, ipb)                                                 \
  for (int64_t i = (int64_t)blockIdx.x * (ipb) + (threadIdx.x >> 5),            \
               i##_end = min((int64_t)(n), ((int64_t)blockIdx.x + 1) * (ipb));  \
       i < i##_end; i += kWarps)

// sites per warp: enough blocks to fill 148 SMs several times over
inline int sites_per_warp(int64_t n) {
  const int64_t ipw = n / (148LL * kWarps * 16);
  return (int)std::max<int64_t>(1, std::min<int64_t>(8, ipw));
}

inline unsigned warp_grid(int64_t n, int ipw) {
  return (unsigned)((n + (int64_t)kWarps * ipw - 1) / ((int64_t)kWarps * ipw));
}

}  // namespace mdg
