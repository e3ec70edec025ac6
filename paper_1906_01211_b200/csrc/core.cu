// core.cu -- context plumbing: errors, launch bookkeeping, deterministic
// reductions, permutation between the caller's order and the device's
// spatially sorted order, Halgren site reduction.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>

#include "common.cuh"

namespace mdg {

[[noreturn]] void throw_error(int code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw_error(MDG_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

static cudaEvent_t pool_event(mdg_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  MDG_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void launch_begin(mdg_ctx* c, const char* name) {
  c->launches++;
  if (c->profile) {
    PendingEvent pe{name, pool_event(c), pool_event(c)};
    MDG_CUDA_CHECK(cudaEventRecord(pe.a, c->stream));
    c->pending.push_back(pe);
  }
}

void launch_end(mdg_ctx* c, const char* name) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw_error(MDG_CUDA, std::string("launch ") + name + ": " +
                                                  cudaGetErrorString(e));
  if (c->profile) MDG_CUDA_CHECK(cudaEventRecord(c->pending.back().b, c->stream));
}

void flush_profile(mdg_ctx* c) {
  if (c->pending.empty()) return;
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  for (auto& pe : c->pending) {
    float ms = 0;
    MDG_CUDA_CHECK(cudaEventElapsedTime(&ms, pe.a, pe.b));
    auto& ent = c->prof[pe.name];
    ent.count++;
    ent.ms += ms;
    c->event_pool.push_back(pe.a);
    c->event_pool.push_back(pe.b);
  }
  c->pending.clear();
}

int64_t sites_per_block(const void* kernel, int64_t n, int bps_cap, int waves_override) {
  static std::mutex mu;
  static std::map<const void*, int> occ;
  static int sms = 0;
  int nb;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (sms == 0) {
      int dev = 0;
      MDG_CUDA_CHECK(cudaGetDevice(&dev));
      MDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    auto it = occ.find(kernel);
    if (it == occ.end()) {
      int v = 0;
      MDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, kBlock, 0));
      it = occ.emplace(kernel, std::max(1, v)).first;
    }
    nb = it->second;
  }
  // 16 waves: long enough per-block site ranges for locality, short enough
  // that the tail of uneven rows does not idle SMs (measured: 1 wave is
  // ~4-7% slower on the multipole/field kernels). MDG_WAVES overrides.
  static const int waves = [] {
    const char* w = std::getenv("MDG_WAVES");
    return w ? std::max(1, std::atoi(w)) : 16;
  }();
  if (bps_cap > 0) nb = std::min(nb, bps_cap);
  const int64_t blocks = (int64_t)sms * nb * (waves_override > 0 ? waves_override : waves);
  return std::max<int64_t>(kWarps, (n + blocks - 1) / blocks);
}

void ensure_partials(mdg_ctx* c, int64_t blocks) {
  if (blocks <= c->partial_blocks) return;
  if (c->partials) cudaFree(c->partials);
  c->partials = nullptr;
  MDG_CUDA_CHECK(cudaMalloc(&c->partials, (size_t)blocks * kRedVals * sizeof(double)));
  c->partial_blocks = blocks;
}

// One block; thread t sums blocks t, t+256, ... then a fixed tree: the
// result does not depend on scheduling.
__global__ void k_finalize(const double* __restrict__ partials, int64_t blocks, int nvals,
                           double scale, double* __restrict__ results, int slot) {
  __shared__ double s[256];
  for (int v = 0; v < nvals; ++v) {
    double acc = 0.0;
    for (int64_t b = threadIdx.x; b < blocks; b += 256) acc += partials[b * kRedVals + v];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) results[slot + v] = s[0] * scale;
    __syncthreads();
  }
}

void finalize_partials(mdg_ctx* c, int64_t blocks, int nvals, int slot, double scale) {
  MDG_LAUNCH(c, "finalize", 1, 256, 0, k_finalize, c->partials, blocks, nvals, scale,
             c->results, slot);
}

void fetch_results(mdg_ctx* c) {
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->h_results, c->results, kResultSlots * sizeof(double),
                                 cudaMemcpyDeviceToHost, c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
}

// ---- permutation kernels --------------------------------------------------

__global__ void k_scatter_scalar(int64_t n, const int32_t* __restrict__ perm,
                                 const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) dst[s] = src[perm[s]];
}

void scatter_sorted_scalar(mdg_ctx* c, const double* d_src, double* d_dst_sorted) {
  MDG_LAUNCH(c, "permute", grid_for(c->n, 256), 256, 0, k_scatter_scalar, c->n, c->d_perm,
             d_src, d_dst_sorted);
}

__global__ void k_gather_vec(int64_t n, const int32_t* __restrict__ perm,
                             const double4* __restrict__ v, double* __restrict__ soa) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) {
    const double4 a = v[s];
    const int64_t o = perm[s];
    soa[o] = a.x;
    soa[n + o] = a.y;
    soa[2 * n + o] = a.z;
  }
}

void gather_vec_to_caller(mdg_ctx* c, const double4* sorted, double* d_dst_soa) {
  MDG_LAUNCH(c, "unpermute", grid_for(c->n, 256), 256, 0, k_gather_vec, c->n, c->d_perm,
             sorted, d_dst_soa);
}

__global__ void k_scatter_vec(int64_t n, const int32_t* __restrict__ perm,
                              const double* __restrict__ soa, double4* __restrict__ v) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) {
    const int64_t o = perm[s];
    v[s] = make_double4(soa[o], soa[n + o], soa[2 * n + o], 0.0);
  }
}

void scatter_vec_from_caller(mdg_ctx* c, const double* d_src_soa, double4* sorted) {
  MDG_LAUNCH(c, "permute", grid_for(c->n, 256), 256, 0, k_scatter_vec, c->n, c->d_perm,
             d_src_soa, sorted);
}

__global__ void k_zero_vec(int64_t n, double4* v) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) v[s] = make_double4(0, 0, 0, 0);
}

void zero_vec(mdg_ctx* c, double4* v) {
  MDG_LAUNCH(c, "zero", grid_for(c->n, 256), 256, 0, k_zero_vec, c->n, v);
}

// ---- Halgren reduced sites --------------------------------------------------
// Bit-identical twin of oracle mdo_reduce_sites and mdg_reduce_sites_host:
// r_red = wrap_into(r_p + f * wrap1(r_i - r_p)), every op separately rounded.
__device__ __forceinline__ double wrap_into_exact(double p, double L) {
  const double k = floor(__ddiv_rn(p, L));
  const double m = __dmul_rn(L, k);
  p = __dsub_rn(p, m);
  if (p >= L) p = 0.0;
  if (p < 0.0) p = 0.0;
  return p;
}

__global__ void k_reduce_sites(int64_t n, Box b, const double4* __restrict__ pos,
                               const int32_t* __restrict__ par, const double* __restrict__ fac,
                               double4* __restrict__ vsite) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 pi = pos[i];
  const int32_t p = par[i];
  if (p == i) {
    vsite[i] = pi;  // w: exclusion group
    return;
  }
  const double4 pp = pos[p];
  const double f = fac[i];
  const double dx = wrap1(__dsub_rn(pi.x, pp.x), b.lx, b.ix, b.hx);
  const double dy = wrap1(__dsub_rn(pi.y, pp.y), b.ly, b.iy, b.hy);
  const double dz = wrap1(__dsub_rn(pi.z, pp.z), b.lz, b.iz, b.hz);
  vsite[i] = make_double4(wrap_into_exact(__dadd_rn(pp.x, __dmul_rn(f, dx)), b.lx),
                          wrap_into_exact(__dadd_rn(pp.y, __dmul_rn(f, dy)), b.ly),
                          wrap_into_exact(__dadd_rn(pp.z, __dmul_rn(f, dz)), b.lz), pi.w);
}

void run_reduce_sites(mdg_ctx* c) {
  Box b = make_box(c->lx, c->ly, c->lz);
  MDG_LAUNCH(c, "reduce_sites", grid_for(c->n, 256), 256, 0, k_reduce_sites, c->n, b, c->pos,
             c->hpar, c->hfac, c->vsite);
}

// ---- system packing: caller-order staging -> sorted device layout -----------
// staging layout: x y z q sig eps r0 heps pol (each n doubles, caller order)
__global__ void k_pack_system(int64_t n, const int32_t* __restrict__ perm,
                              const double* __restrict__ st, double4* __restrict__ pos,
                              double4* __restrict__ vsite, double4* __restrict__ vdwp,
                              double2* __restrict__ polp, double4* __restrict__ pq4,
                              const int32_t* __restrict__ vtype) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t o = perm[s];
  const double x = st[o], y = st[n + o], z = st[2 * n + o];
  const double q = st[3 * n + o];
  // w of pos / vsite: the site's exclusion group (identity until
  // mdg_topology_upload; see set_groups), read by the pair prologues
  const int32_t t = vtype ? vtype[s] : 0;
  pos[s] = make_double4(x, y, z, group_bits((int32_t)s, t));
  vsite[s] = make_double4(x, y, z, group_bits((int32_t)s, t));
  vdwp[s] = make_double4(st[4 * n + o], sqrt(st[5 * n + o]), st[6 * n + o], sqrt(st[7 * n + o]));
  const double pol = st[8 * n + o];
  const double pd = cbrt(sqrt(pol));
  polp[s] = make_double2(pol, pd);
  pq4[s] = make_double4(pol, pd, q, 1.0 / pd);  // w: 1/pdamp (Thole u = r ipd_i ipd_j)
}

void pack_system(mdg_ctx* c) {
  MDG_LAUNCH(c, "pack_system", grid_for(c->n, 256), 256, 0, k_pack_system, c->n, c->d_perm,
             c->d_stage, c->pos, c->vsite, c->vdwp, c->polp, c->pq4,
             c->n_vtypes ? c->vtype : nullptr);
}

// staging: x y z (caller order); keeps charges
__global__ void k_pack_positions(int64_t n, const int32_t* __restrict__ perm,
                                 const double* __restrict__ st, double4* __restrict__ pos,
                                 double4* __restrict__ vsite, int copy_vsite) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t o = perm[s];
  const double x = st[o], y = st[n + o], z = st[2 * n + o];
  pos[s].x = x;
  pos[s].y = y;
  pos[s].z = z;
  if (copy_vsite) vsite[s] = make_double4(x, y, z, pos[s].w);
}

// position contract 0 <= r < L on the staged caller-order arrays: the lowest
// offending caller index goes to flag[6] (0x7f7f7f7f: none)
__global__ void k_check_box(int64_t n, const double* __restrict__ st, double lx, double ly,
                            double lz, int32_t* __restrict__ flag) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= n) return;
  const double x = st[o], y = st[n + o], z = st[2 * n + o];
  const bool ok = (x >= 0.0) & (x < lx) & (y >= 0.0) & (y < ly) & (z >= 0.0) & (z < lz);
  if (!ok) atomicMin(&flag[6], (int32_t)o);
}

int64_t check_box_staged(mdg_ctx* c, int64_t count) {
  const int64_t n = count >= 0 ? count : c->n;
  MDG_CUDA_CHECK(cudaMemsetAsync(c->d_flag + 6, 0x7f, sizeof(int32_t), c->stream));
  MDG_LAUNCH(c, "check_box", grid_for(n, 256), 256, 0, k_check_box, n, c->d_stage, c->lx,
             c->ly, c->lz, c->d_flag);
  int32_t bad = 0;
  MDG_CUDA_CHECK(cudaMemcpyAsync(&bad, c->d_flag + 6, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return bad == 0x7f7f7f7f ? -1 : bad;
}

__global__ void k_set_groups(int64_t n, const int32_t* __restrict__ mol,
                             const int32_t* __restrict__ vtype, double4* __restrict__ pos,
                             double4* __restrict__ vsite) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int32_t t = vtype ? vtype[s] : 0;
  pos[s].w = group_bits(mol[s], t);
  vsite[s].w = group_bits(mol[s], t);
}

__global__ void k_vtab(int nt, const int32_t* __restrict__ rep, const double4* __restrict__ vdwp,
                       const double4* __restrict__ pq4, double4* __restrict__ vtab,
                       double4* __restrict__ ptab) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nt) {
    vtab[t] = vdwp[rep[t]];
    ptab[t] = pq4[rep[t]];
  }
}

// rep[t] = a sorted-order site of type t; vtype already on the device.
// vtab / ptab are bit copies of those sites' vdwp / pq4 records (the values a
// gather would read).
void set_vdw_types(mdg_ctx* c, const std::vector<int32_t>& rep) {
  c->n_vtypes = (int)rep.size();
  if (rep.empty()) return;
  int32_t* d_rep = c->d_idx;  // staging (n >= n_vtypes)
  MDG_CUDA_CHECK(cudaMemcpyAsync(d_rep, rep.data(), rep.size() * 4, cudaMemcpyHostToDevice,
                                 c->stream));
  MDG_LAUNCH(c, "vtab", 1, kMaxVdwTypes, 0, k_vtab, (int)rep.size(), d_rep, c->vdwp, c->pq4,
             c->vtab, c->ptab);
}

void set_groups(mdg_ctx* c) {
  MDG_LAUNCH(c, "set_groups", grid_for(c->n, 256), 256, 0, k_set_groups, c->n, c->mol,
             c->n_vtypes ? c->vtype : nullptr, c->pos,
             c->vsite);
}

__global__ void k_copy_vsite(int64_t n, const double4* __restrict__ pos, double4* __restrict__ vsite) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) vsite[s] = pos[s];
}

void pack_positions(mdg_ctx* c, int64_t count) {
  // count >= 0: the owned sites (sorted first, and first in caller order),
  // staged with stride count; the halo comes from the group's exchange
  const int64_t n = count >= 0 ? count : c->n;
  MDG_LAUNCH(c, "pack_positions", grid_for(n, 256), 256, 0, k_pack_positions, n, c->d_perm,
             c->d_stage, c->pos, c->vsite, c->has_hred ? 0 : 1);
  if (c->has_hred) run_reduce_sites(c);
}

// ---- halo exchange: pack / unpack 3 doubles per listed caller-order site ----
__global__ void k_vec_pack(int64_t count, const int32_t* __restrict__ sites,
                           const int32_t* __restrict__ iperm, const double4* __restrict__ v,
                           double* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double4 a = v[iperm[sites[k]]];
  out[3 * k] = a.x;
  out[3 * k + 1] = a.y;
  out[3 * k + 2] = a.z;
}

__global__ void k_vec_unpack(int64_t count, const int32_t* __restrict__ sites,
                             const int32_t* __restrict__ iperm, const double* __restrict__ in,
                             double4* __restrict__ v) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  double4* a = v + iperm[sites[k]];
  a->x = in[3 * k];
  a->y = in[3 * k + 1];
  a->z = in[3 * k + 2];
}

double4* vec_by_id(mdg_ctx* c, int vec_id) {
  switch (vec_id) {
    case MDG_VEC_POS: return c->pos;
    case MDG_VEC_MU: return c->mu;
    case MDG_VEC_P: return c->cg_p;
    case MDG_VEC_FORCE: return c->force;
    case MDG_VEC_TORQUE: return c->torque;
    case MDG_VEC_EPERM: return c->eperm;
    default: throw_error(MDG_CONTRACT, "unknown vector id");
  }
}

void vec_pack(mdg_ctx* c, int vec_id, const int32_t* d_sites, int64_t count, double* d_out) {
  if (count <= 0) return;
  MDG_LAUNCH(c, "halo_pack", grid_for(count, 256), 256, 0, k_vec_pack, count, d_sites, c->d_iperm,
             vec_by_id(c, vec_id), d_out);
}

void vec_unpack(mdg_ctx* c, int vec_id, const int32_t* d_sites, int64_t count,
                const double* d_in) {
  if (count <= 0) return;
  MDG_LAUNCH(c, "halo_unpack", grid_for(count, 256), 256, 0, k_vec_unpack, count, d_sites,
             c->d_iperm, d_in, vec_by_id(c, vec_id));
  if (vec_id == MDG_VEC_POS) refresh_vsites(c);
}

void refresh_vsites(mdg_ctx* c) {
  if (c->has_hred) run_reduce_sites(c);
  else MDG_LAUNCH(c, "copy_vsite", grid_for(c->n, 256), 256, 0, k_copy_vsite, c->n, c->pos,
                  c->vsite);
}

// -E_pol = 1/2 sum mu . E_perm ; results[slot] = -0.5 * electric * sum
__global__ void __launch_bounds__(kBlock) k_dot4(int64_t n, const double4* __restrict__ a,
                                                 const double4* __restrict__ b,
                                                 double* __restrict__ partials) {
  const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  double acc[1] = {0.0};
  if (i < n) {
    const double4 x = a[i], y = b[i];
    acc[0] = x.x * y.x + x.y * y.y + x.z * y.z;
  }
  block_store_partials<1>(acc, partials);
}

void polar_energy(mdg_ctx* c, double electric, int slot) {
  const int64_t blocks = grid_for(c->n_own);
  ensure_partials(c, blocks);
  MDG_LAUNCH(c, "dot", (unsigned)blocks, kBlock, 0, k_dot4, c->n_own, c->mu, c->eperm,
             c->partials);
  finalize_partials(c, blocks, 1, slot, -0.5 * electric);
}

}  // namespace mdg
