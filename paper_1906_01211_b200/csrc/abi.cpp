// abi.cpp -- extern "C" boundary (include/mdg.h): validation with the
// reference's contract checks and error taxonomy, host<->device staging,
// spatial sort, list import/export in the reference NeighborTable layout,
// and the fused steps. No kernels here; they live in the .cu files.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <numeric>
#include <string>
#include <vector>

#include "mdg_internal.h"

using mdg::throw_error;

namespace {

thread_local std::string g_err;

std::atomic<uint64_t> g_api_seq{0};  // API calls so far (process-wide)

template <class F>
int guard(F&& f) {
  g_api_seq.fetch_add(1, std::memory_order_relaxed);
  try {
    f();
    return MDG_OK;
  } catch (const mdg::Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return MDG_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MDG_CUDA;
  }
}

void need(bool ok, const char* msg) {
  if (!ok) throw_error(MDG_CONTRACT, msg);
}

void need_ctx(mdg_ctx* c) { need(c != nullptr, "null context"); }

void need_system(mdg_ctx* c) {
  need_ctx(c);
  need(c->has_system, "no system uploaded");
}

template <class T>
void dalloc(T** p, size_t count) {
  MDG_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
}

void set_device(mdg_ctx* c) { MDG_CUDA_CHECK(cudaSetDevice(c->device)); }

mdg::DevList& need_list(mdg_ctx* c, int list_id) {
  need(list_id >= 0 && list_id < MDG_MAX_LISTS, "list id out of range");
  mdg::DevList& L = c->lists[list_id];
  need(L.valid, "neighbour list not built");
  return L;
}

// proj/src/kernels_impl.hpp:14-16
void need_kernel_cutoff(const mdg::DevList& L, double cutoff) {
  need(cutoff > 0 && cutoff <= L.cutoff,
       "kernel: cutoff must be positive and within the list cutoff");
}

// Morton interleave of three 21-bit cell coordinates
uint64_t spread3(uint64_t v) {
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

// Spatial order: Morton order over ~2 A cells, stable in the caller's index,
// so every 32-site group (one warp) is a compact blob of space.
void spatial_sort(mdg_ctx* c, const double* x, const double* y, const double* z) {
  const int64_t n = c->n;
  const int nx = std::max(1, (int)(c->lx / 2.0)), ny = std::max(1, (int)(c->ly / 2.0)),
            nz = std::max(1, (int)(c->lz / 2.0));
  std::vector<uint64_t> key(n);
  for (int64_t i = 0; i < n; ++i) {
    const int cx = std::min(nx - 1, (int)(x[i] / c->lx * nx));
    const int cy = std::min(ny - 1, (int)(y[i] / c->ly * ny));
    const int cz = std::min(nz - 1, (int)(z[i] / c->lz * nz));
    key[i] = spread3(cx) | spread3(cy) << 1 | spread3(cz) << 2;
  }
  c->perm.resize(n);
  std::iota(c->perm.begin(), c->perm.end(), 0);
  // owned sites first (rows), then the halo; each part in Morton order
  auto by_key = [&](int32_t a, int32_t b) { return key[a] < key[b]; };
  std::stable_sort(c->perm.begin(), c->perm.begin() + c->n_own, by_key);
  std::stable_sort(c->perm.begin() + c->n_own, c->perm.end(), by_key);
  c->iperm.resize(n);
  for (int64_t s = 0; s < n; ++s) c->iperm[c->perm[s]] = (int32_t)s;
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_perm, c->perm.data(), n * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, c->stream));
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_iperm, c->iperm.data(), n * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, c->stream));
}

// Host-side copies of the per-step vectors (24 B/site each way) run on up to
// 8 threads: a single-threaded memcpy into pinned memory was most of the
// end-to-end overhead at 10^6 sites.
void host_parallel(int64_t n, const std::function<void(int64_t, int64_t)>& f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t T = std::min<int64_t>(std::min<unsigned>(8, hw), std::max<int64_t>(1, n >> 16));
  if (T <= 1) {
    f(0, n);
    return;
  }
  const int64_t chunk = (n + T - 1) / T;
  std::vector<std::thread> th;
  for (int64_t t = 1; t < T; ++t) {
    const int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b < e) th.emplace_back(f, b, e);
  }
  f(0, std::min(n, chunk));
  for (auto& x : th) x.join();
}

static bool is_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Copy caller arrays into the pinned stage and upload them (or, when every
// array is page-locked, DMA them directly). With `box`, the first three
// arrays are positions and are checked to lie in [0, L) (the ParticleSystem
// contract, proj/src/system.cpp): page-locked positions on the device after
// the DMA (one pass over 24 B/site in HBM instead of a host pass competing
// with the DMA for the same pages), staged ones on the host during the copy.
// Returns with the caller's arrays no longer in use.
// (count >= 0: the first `count` caller-order sites only, staged with stride
// count -- the owned sites of a domain)
void stage_in(mdg_ctx* c, const std::vector<const double*>& arrays, const double* box = nullptr,
              int64_t count = -1) {
  const int64_t n = count >= 0 ? count : c->n;
  bool pinned = true;
  for (const double* a : arrays) pinned = pinned && is_pinned(a);
  if (pinned) {
    for (size_t a = 0; a < arrays.size(); ++a)
      MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_stage + a * n, arrays[a], n * sizeof(double),
                                     cudaMemcpyHostToDevice, c->stream));
    if (box) {  // box is the context's (c->lx, c->ly, c->lz)
      need(mdg::check_box_staged(c, n) < 0, "ParticleSystem: position outside the box");
    } else {
      MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
    return;
  }
  std::atomic<bool> bad{false};
  host_parallel(n, [&](int64_t b, int64_t e) {
    for (size_t a = 0; a < arrays.size(); ++a) {
      const double* src = arrays[a];
      std::memcpy(c->h_stage + a * n + b, src + b, (e - b) * sizeof(double));
      if (box && a < 3) {
        const double L = box[a];
        bool ok = true;
        for (int64_t i = b; i < e; ++i) ok &= (src[i] >= 0.0) & (src[i] < L);
        if (!ok) bad = true;
      }
    }
  });
  need(!bad, "ParticleSystem: position outside the box");
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_stage, c->h_stage, arrays.size() * n * sizeof(double),
                                 cudaMemcpyHostToDevice, c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));  // h_stage free for the next call
}

// sorted double4 vector -> caller-order SoA host arrays (NULL entries skipped)
void vec_out(mdg_ctx* c, const double4* v, double* ox, double* oy, double* oz) {
  if (!ox && !oy && !oz) return;
  const int64_t n = c->n;
  mdg::gather_vec_to_caller(c, v, c->d_stage);
  double* outs[3] = {ox, oy, oz};
  bool pinned = true;
  for (double* o : outs) pinned = pinned && (!o || is_pinned(o));
  if (pinned) {
    for (int a = 0; a < 3; ++a)
      if (outs[a])
        MDG_CUDA_CHECK(cudaMemcpyAsync(outs[a], c->d_stage + a * n, n * sizeof(double),
                                       cudaMemcpyDeviceToHost, c->stream));
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return;
  }
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->h_stage, c->d_stage, 3 * n * sizeof(double),
                                 cudaMemcpyDeviceToHost, c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  host_parallel(n, [&](int64_t b, int64_t e) {
    for (int a = 0; a < 3; ++a)
      if (outs[a]) std::memcpy(outs[a] + b, c->h_stage + a * n + b, (e - b) * sizeof(double));
  });
}

void vec_in(mdg_ctx* c, const double* ix, const double* iy, const double* iz, double4* v) {
  stage_in(c, {ix, iy, iz});
  mdg::scatter_vec_from_caller(c, c->d_stage, v);
}

void sym_virial(const double* s6, double* w9) {
  // s6: xx xy xz yy yz zz
  w9[0] = s6[0]; w9[1] = s6[1]; w9[2] = s6[2];
  w9[3] = s6[1]; w9[4] = s6[3]; w9[5] = s6[4];
  w9[6] = s6[2]; w9[7] = s6[4]; w9[8] = s6[5];
}

int64_t pad_count(int64_t n, int64_t m) { return (n + m - 1) & ~(m - 1); }

}  // namespace

namespace mdg {
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace mdg

extern "C" {

const char* mdg_last_error(void) { return g_err.c_str(); }

int mdg_version(void) { return 1; }

int mdg_ctx_create(mdg_ctx** out, int device, int64_t n_capacity, int32_t max_pairs_per_atom) {
  return guard([&] {
    need(out != nullptr, "null output pointer");
    need(n_capacity > 0 && n_capacity < (int64_t)1 << 30, "n_capacity out of range");
    auto* c = new mdg_ctx();
    *out = nullptr;
    try {
      c->device = device;
      if (const char* d = getenv("MDG_DETERMINISTIC")) c->deterministic = atoi(d) != 0;
      if (const char* o = getenv("MDG_OVERLAP")) c->overlap = atoi(o) != 0;
      if (const char* o = getenv("MDG_CLUSTER_MATVEC")) c->cluster_matvec = atoi(o) != 0;
      if (const char* o = getenv("MDG_CLUSTER_HALGREN")) c->cluster_halgren = atoi(o) != 0;
      set_device(c);
      c->n_cap = n_capacity;
      c->max_pairs = max_pairs_per_atom > 0 ? max_pairs_per_atom : 2 * MDG_MAX_NEIGHBORS;
      {
        // the context stream carries the step's critical path (field -> PCG);
        // it outranks the aux stream (Halgren, multipoles) at block dispatch
        int lo = 0, hi = 0;
        MDG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        MDG_CUDA_CHECK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi));
      }
      const size_t n = (size_t)n_capacity;
      dalloc(&c->d_perm, n);
      dalloc(&c->d_iperm, n);
      dalloc(&c->d_idx, n);
      dalloc(&c->pos, n);
      dalloc(&c->vsite, n);
      dalloc(&c->vdwp, n);
      dalloc(&c->vtype, n);
      dalloc(&c->vtab, (size_t)kMaxVdwTypes);
      dalloc(&c->ptab, (size_t)kMaxVdwTypes);
      dalloc(&c->polp, n);
      dalloc(&c->mol, n);
      dalloc(&c->hpar, n);
      dalloc(&c->hfac, n);
      dalloc(&c->child_start, n + 1);
      dalloc(&c->child, n);
      dalloc(&c->mp, 3 * n);
      dalloc(&c->cell_of, n);
      dalloc(&c->cell_atoms, n);
      dalloc(&c->d_flag, 8);
      MDG_CUDA_CHECK(cudaMemset(c->d_flag, 0, 8 * sizeof(int32_t)));
      for (double4** v : {&c->force, &c->force2, &c->torque, &c->field, &c->eperm, &c->mu,
                          &c->cg_r, &c->cg_z, &c->cg_p, &c->cg_q, &c->vin, &c->pq4})
        dalloc(v, n);
      dalloc(&c->results, mdg::kResultSlots);
      MDG_CUDA_CHECK(cudaMemset(c->results, 0, mdg::kResultSlots * sizeof(double)));
      MDG_CUDA_CHECK(cudaMallocHost(&c->h_results, mdg::kResultSlots * sizeof(double)));
      MDG_CUDA_CHECK(cudaHostAlloc(&c->h_warn, sizeof(int32_t), cudaHostAllocMapped));
      *c->h_warn = 0;
      MDG_CUDA_CHECK(cudaHostGetDevicePointer(&c->d_warn, c->h_warn, 0));
      c->stage_bytes = 12 * n * sizeof(double);
      MDG_CUDA_CHECK(cudaMallocHost(&c->h_stage, c->stage_bytes));
      dalloc(&c->d_stage, 12 * n);
      mdg::ensure_partials(c, mdg::grid_for(n_capacity));
    } catch (...) {
      mdg_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

int mdg_ctx_destroy(mdg_ctx* c) {
  if (!c) return MDG_OK;
  if (c->group) {  // the group still references this context (and owns its stream)
    mdg::set_error("mdg_ctx_destroy: context is in a domain group; call mdg_group_destroy first");
    return MDG_CONTRACT;
  }
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->aux_stream) cudaStreamSynchronize(c->aux_stream);
  void* ptrs[] = {c->d_perm, c->d_iperm, c->d_idx, c->pos, c->vsite, c->vdwp, c->vtype, c->vtab, c->ptab, c->polp, c->mol, c->hpar, c->hfac,
                  c->child_start, c->child, c->mp, c->frame, c->mploc, c->fbuf, c->fref_start,
                  c->excl_start, c->excl, c->vel, c->fbond, c->bond_ij, c->bond_par, c->angle_ijk,
                  c->angle_par,
                  c->fref, c->cell_of, c->cell_start, c->cell_fill,
                  c->cell_atoms, c->d_flag, c->force, c->force2, c->torque, c->field, c->eperm,
                  c->mu, c->cg_r, c->cg_z, c->cg_p, c->cg_q, c->vin, c->pq4, c->partials,
                  c->results,
                  c->d_stage, c->dd_sites, c->dd_flags, c->dd_nsel, c->dd_tmp,
                  c->aspc_hist};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& L : c->lists) {
    if (L.nbr) cudaFree(L.nbr);
    if (L.cnt) cudaFree(L.cnt);
    if (L.ref0) cudaFree(L.ref0);
    for (void* p : {(void*)L.inner.nbr, (void*)L.inner.cnt, (void*)L.inner.ref, (void*)L.inner.flag,
                     (void*)L.inner.gen, (void*)L.inner.uidx, (void*)L.inner.ucnt,
                     (void*)L.inner.ugen})
      if (p) cudaFree(p);
    if (L.inner.hcuts) cudaFreeHost(L.inner.hcuts);
  }
  if (c->plist.nbr) cudaFree(c->plist.nbr);
  if (c->plist.cnt) cudaFree(c->plist.cnt);
  if (c->plist.trr) cudaFree(c->plist.trr);
  if (c->plist.ucnt) cudaFree(c->plist.ucnt);
  if (c->plist.ugen) cudaFree(c->plist.ugen);
  if (c->plist.cmap) cudaFree(c->plist.cmap);
  if (c->plist.cst) cudaFree(c->plist.cst);
  if (c->h_results) cudaFreeHost(c->h_results);
  if (c->h_warn) cudaFreeHost(c->h_warn);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto& pe : c->pending) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->timer_a) cudaEventDestroy(c->timer_a);
  if (c->timer_b) cudaEventDestroy(c->timer_b);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  mdg::pme_free(c);
  mdg::pcg_graph_forget(c);
  if (c->aux_partials) cudaFree(c->aux_partials);
  for (cudaEvent_t e : {c->ev_fork, c->ev_tpre, c->ev_join})
    if (e) cudaEventDestroy(e);
  delete c;
  return MDG_OK;
}

int mdg_ctx_synchronize(mdg_ctx* c) {
  return guard([&] {
    need_ctx(c);
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

void* mdg_ctx_stream(mdg_ctx* c) { return c ? (void*)c->stream : nullptr; }

int mdg_system_upload(mdg_ctx* c, int64_t n, double lx, double ly, double lz, const double* x,
                      const double* y, const double* z, const double* charge,
                      const double* lj_sigma, const double* lj_epsilon, const double* hal_r0,
                      const double* hal_epsilon, const double* polarizability) {
  return mdg_system_upload_owned(c, n, n, n, lx, ly, lz, x, y, z, charge, lj_sigma, lj_epsilon,
                                 hal_r0, hal_epsilon, polarizability);
}

// Distinct (sigma, eps_lj, r0, eps_hal, charge, polarizability) tuples (bitwise) in sorted order:
// vtype[s] = type of sorted site s, rep[t] = first sorted site of type t.
// False when there are more than kMaxVdwTypes tuples (per-site gathers then).
static bool assign_vdw_types(const std::vector<int32_t>& perm, const double* sig,
                             const double* eps, const double* r0, const double* eh,
                             const double* q, const double* pol, std::vector<int32_t>& vtype,
                             std::vector<int32_t>& rep) {
  std::map<std::array<uint64_t, 6>, int32_t> types;
  for (size_t s = 0; s < vtype.size(); ++s) {
    const int64_t o = perm[s];
    const double v[6] = {sig[o], eps[o], r0[o], eh[o], q[o], pol[o]};
    std::array<uint64_t, 6> key;
    std::memcpy(key.data(), v, sizeof v);
    auto it = types.find(key);
    if (it == types.end()) {
      if ((int)types.size() == kMaxVdwTypes) return false;
      it = types.emplace(key, (int32_t)types.size()).first;
      rep.push_back((int32_t)s);
    }
    vtype[s] = it->second;
  }
  return true;
}

int mdg_system_upload_owned(mdg_ctx* c, int64_t n, int64_t n_owned, int64_t n_global,
                            double lx, double ly, double lz, const double* x, const double* y,
                            const double* z, const double* charge, const double* lj_sigma,
                            const double* lj_epsilon, const double* hal_r0,
                            const double* hal_epsilon, const double* polarizability) {
  return guard([&] {
    need_ctx(c);
    set_device(c);
    need(n_owned >= 1 && n_owned <= n, "system: owned count must be in [1, n]");
    need(n_global >= n, "system: global count must cover the local sites");
    c->n_own = n_owned;
    c->n_global = n_global;
    // OrthorhombicBox::validate (proj/include/mdvec/pbc.hpp:14-19)
    need(lx > 0 && ly > 0 && lz > 0 && std::isfinite(lx) && std::isfinite(ly) &&
             std::isfinite(lz),
         "OrthorhombicBox: edges must be positive and finite");
    need(n >= 1 && n <= c->n_cap, "ParticleSystem: site count outside the context capacity");
    need(x && y && z && charge && lj_sigma && lj_epsilon && hal_r0 && hal_epsilon &&
             polarizability,
         "ParticleSystem: null array");
    // proj/src/system.cpp:18-27
    const double L[3] = {lx, ly, lz};
    const double* p[3] = {x, y, z};
    for (int a = 0; a < 3; ++a)
      for (int64_t i = 0; i < n; ++i)
        need(p[a][i] >= 0.0 && p[a][i] < L[a], "ParticleSystem: position outside the box");
    c->n = n;
    c->lx = lx;
    c->ly = ly;
    c->lz = lz;
    for (auto& Lst : c->lists) Lst.valid = false;
    c->has_mpoles = c->has_hred = c->has_mol = c->has_frames = false;
    c->mol_sorted = false;
    c->fout[0] = c->fout[1] = c->fout[2] = nullptr;  // sized for the old system
    spatial_sort(c, x, y, z);
    stage_in(c, {x, y, z, charge, lj_sigma, lj_epsilon, hal_r0, hal_epsilon, polarizability});
    // vdW parameter types (bitwise-distinct tuples, in sorted order)
    std::vector<int32_t> vtype(n), rep;
    c->n_vtypes = 0;
    if (assign_vdw_types(c->perm, lj_sigma, lj_epsilon, hal_r0, hal_epsilon, charge,
                         polarizability, vtype, rep) &&
        !mdg::env_int("MDG_NO_VDW_TYPES", 0)) {
      MDG_CUDA_CHECK(cudaMemcpyAsync(c->vtype, vtype.data(), n * 4, cudaMemcpyHostToDevice,
                                     c->stream));
      c->n_vtypes = (int)rep.size();
    } else {
      rep.clear();
    }
    mdg::pack_system(c);
    mdg::set_vdw_types(c, rep);
    // identity topology: every site its own group, no reduction
    std::vector<int32_t> ident(n);
    std::iota(ident.begin(), ident.end(), 0);
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->mol, ident.data(), n * 4, cudaMemcpyHostToDevice,
                                   c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->hpar, ident.data(), n * 4, cudaMemcpyHostToDevice,
                                   c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(c->mp, 0, 3 * n * sizeof(double4), c->stream));
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    c->has_system = true;
  });
}

int mdg_set_ewald_recip(mdg_ctx* c, int k1, int k2, int k3, int order) {
  return guard([&] {
    need_ctx(c);
    if (k1 <= 0) {
      c->pol_recip = mdg::PolarRecip{};
      return;
    }
    need(order >= 5 && order <= 10, "ewald_recip: B-spline order must be 5..10");
    need(k2 > 0 && k3 > 0 && k1 >= order && k2 >= order && k3 >= order,
         "ewald_recip: grid smaller than the order");
    c->pol_recip.k1 = k1;
    c->pol_recip.k2 = k2;
    c->pol_recip.k3 = k3;
    c->pol_recip.order = order;
  });
}

int mdg_set_deterministic(mdg_ctx* c, int on) {
  return guard([&] {
    need_ctx(c);
    c->deterministic = on != 0;
  });
}

int mdg_host_alloc(void** ptr, int64_t bytes) {
  return guard([&] {
    need(ptr != nullptr && bytes > 0, "host_alloc: bad arguments");
    MDG_CUDA_CHECK(cudaHostAlloc(ptr, (size_t)bytes, cudaHostAllocPortable));
  });
}

int mdg_host_free(void* ptr) {
  return guard([&] {
    if (ptr) MDG_CUDA_CHECK(cudaFreeHost(ptr));
  });
}

int mdg_set_overlap(mdg_ctx* c, int on) {
  return guard([&] {
    need_ctx(c);
    c->overlap = on != 0;
  });
}

int mdg_set_cluster_matvec(mdg_ctx* c, int on) {
  return guard([&] {
    need_ctx(c);
    c->cluster_matvec = on != 0;
  });
}

int mdg_set_cluster_halgren(mdg_ctx* c, int on) {
  return guard([&] {
    need_ctx(c);
    c->cluster_halgren = on != 0;
  });
}

int mdg_vec_pack(mdg_ctx* c, int vec_id, const int32_t* sites, int64_t count, double* out) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(count >= 0 && count <= c->n, "vec_pack: count out of range");
    if (count == 0) return;
    for (int64_t k = 0; k < count; ++k)
      need(sites[k] >= 0 && sites[k] < c->n, "vec_pack: site out of range");
    int32_t* hidx = reinterpret_cast<int32_t*>(c->h_stage + 3 * count);
    std::memcpy(hidx, sites, count * sizeof(int32_t));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_idx, hidx, count * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, c->stream));
    mdg::vec_pack(c, vec_id, c->d_idx, count, c->d_stage);
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->h_stage, c->d_stage, 3 * count * sizeof(double),
                                   cudaMemcpyDeviceToHost, c->stream));
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    std::memcpy(out, c->h_stage, 3 * count * sizeof(double));
  });
}

int mdg_vec_unpack(mdg_ctx* c, int vec_id, const int32_t* sites, int64_t count,
                   const double* in) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(count >= 0 && count <= c->n, "vec_unpack: count out of range");
    if (count == 0) return;
    for (int64_t k = 0; k < count; ++k)
      need(sites[k] >= 0 && sites[k] < c->n, "vec_unpack: site out of range");
    int32_t* hidx = reinterpret_cast<int32_t*>(c->h_stage + 3 * count);
    std::memcpy(c->h_stage, in, 3 * count * sizeof(double));
    std::memcpy(hidx, sites, count * sizeof(int32_t));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_idx, hidx, count * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->d_stage, c->h_stage, 3 * count * sizeof(double),
                                   cudaMemcpyHostToDevice, c->stream));
    mdg::vec_unpack(c, vec_id, c->d_idx, count, c->d_stage);
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int mdg_vec_pack_dev(mdg_ctx* c, int vec_id, const int32_t* d_sites, int64_t count,
                     double* d_out) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(count >= 0 && count <= c->n, "vec_pack_dev: count out of range");
    mdg::vec_pack(c, vec_id, d_sites, count, d_out);
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int mdg_vec_unpack_dev(mdg_ctx* c, int vec_id, const int32_t* d_sites, int64_t count,
                       const double* d_in) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(count >= 0 && count <= c->n, "vec_unpack_dev: count out of range");
    mdg::vec_unpack(c, vec_id, d_sites, count, d_in);
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int mdg_positions_upload(mdg_ctx* c, const double* x, const double* y, const double* z) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(x && y && z, "null position array");
    const double L[3] = {c->lx, c->ly, c->lz};
    stage_in(c, {x, y, z}, L);
    mdg::pack_positions(c);
  });
}

int mdg_positions_upload_owned(mdg_ctx* c, const double* x, const double* y, const double* z) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(x && y && z, "null position array");
    const double L[3] = {c->lx, c->ly, c->lz};
    stage_in(c, {x, y, z}, L, c->n_own);
    mdg::pack_positions(c, c->n_own);
  });
}

int mdg_topology_upload(mdg_ctx* c, const int32_t* molecule, const int32_t* hred_parent,
                        const double* hred_factor) {
  return guard([&] {
    need_system(c);
    set_device(c);
    const int64_t n = c->n;
    std::vector<int32_t> mol(n), par(n);
    std::vector<double> fac(n, 1.0);
    for (int64_t s = 0; s < n; ++s) {
      const int32_t o = c->perm[s];
      mol[s] = molecule ? molecule[o] : o;
      if (hred_parent) {
        const int32_t po = hred_parent[o];
        need(po >= 0 && po < n, "topology: reduction parent out of range");
        par[s] = c->iperm[po];
        fac[s] = hred_factor ? hred_factor[o] : 1.0;
      } else {
        par[s] = (int32_t)s;
      }
    }
    // same-molecule partners per site (CSR, sorted indices): PME removes these
    // pairs from the reciprocal sum
    {
      std::map<int32_t, std::vector<int32_t>> groups;
      for (int64_t s = 0; s < n; ++s) groups[mol[s]].push_back((int32_t)s);
      std::vector<int32_t> xs(n + 1, 0), xl;
      for (int64_t s = 0; s < n; ++s) xs[s + 1] = (int32_t)groups[mol[s]].size() - 1;
      for (int64_t s = 0; s < n; ++s) xs[s + 1] += xs[s];
      xl.resize(std::max<int32_t>(xs[n], 1));
      for (int64_t s = 0; s < n; ++s) {
        int32_t k = xs[s];
        for (int32_t t : groups[mol[s]])
          if (t != s) xl[k++] = t;
      }
      if (c->excl) cudaFree(c->excl);
      c->excl = nullptr;
      if (!c->excl_start)
        MDG_CUDA_CHECK(cudaMalloc(&c->excl_start, ((size_t)c->n_cap + 1) * sizeof(int32_t)));
      MDG_CUDA_CHECK(cudaMalloc(&c->excl, xl.size() * sizeof(int32_t)));
      MDG_CUDA_CHECK(cudaMemcpy(c->excl_start, xs.data(), (n + 1) * sizeof(int32_t),
                                cudaMemcpyHostToDevice));
      MDG_CUDA_CHECK(cudaMemcpy(c->excl, xl.data(), xl.size() * sizeof(int32_t),
                                cudaMemcpyHostToDevice));
    }
    // children CSR (sorted indices) for the chain rule; a parent must be its own parent
    std::vector<int32_t> start(n + 1, 0), child;
    for (int64_t s = 0; s < n; ++s)
      if (par[s] != s) {
        need(par[par[s]] == par[s], "topology: reduction parents must not be reduced");
        start[par[s] + 1]++;
      }
    for (int64_t s = 0; s < n; ++s) start[s + 1] += start[s];
    child.resize(std::max<int32_t>(start[n], 1));
    std::vector<int32_t> fill(start.begin(), start.end() - 1);
    for (int64_t s = 0; s < n; ++s)
      if (par[s] != s) child[fill[par[s]]++] = (int32_t)s;
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->mol, mol.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->hpar, par.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->hfac, fac.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->child_start, start.data(), (n + 1) * 4,
                                   cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->child, child.data(), child.size() * 4,
                                   cudaMemcpyHostToDevice, c->stream));
    c->has_mol = molecule != nullptr;
    c->has_hred = hred_parent != nullptr;
    mdg::set_groups(c);
    if (c->has_hred) mdg::run_reduce_sites(c);
    // molecule-keyed site order (a domain's owned and halo parts each): a
    // molecule's sites consecutive, so the 3-site clusters are water
    // molecules (cluster.cu)
    static const int mol_order = mdg::env_int("MDG_MOL_ORDER", 1);
    if (molecule && mol_order && !c->group && mdg::mol_order_fits(c)) {
      std::unordered_map<int32_t, int32_t> first;  // molecule -> lowest caller index
      first.reserve((size_t)n);
      for (int64_t s = 0; s < n; ++s) {
        auto it = first.emplace(mol[s], c->perm[s]).first;
        it->second = std::min(it->second, c->perm[s]);
      }
      std::vector<int32_t> rep(n);
      for (int64_t s = 0; s < n; ++s) rep[s] = c->iperm[first[mol[s]]];
      int32_t* d_rep = nullptr;
      MDG_CUDA_CHECK(cudaMalloc(&d_rep, (size_t)n * sizeof(int32_t)));
      MDG_CUDA_CHECK(cudaMemcpyAsync(d_rep, rep.data(), (size_t)n * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, c->stream));
      mdg::resort_sites(c, d_rep);  // synchronises the stream
      MDG_CUDA_CHECK(cudaFree(d_rep));
    }
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int mdg_frames_upload(mdg_ctx* c, const int32_t* frame_type, const int32_t* zatom,
                      const int32_t* xatom, const double* dipole, const double* quadrupole) {
  return guard([&] {
    need_system(c);
    set_device(c);
    const int64_t n = c->n;
    if (!frame_type) {
      c->has_frames = false;
      return;
    }
    need(zatom && xatom, "frames: zatom and xatom are required");
    std::vector<int32_t> fr(4 * n, 0);
    std::vector<int32_t> cnt(n + 1, 0);
    bool any = false;
    for (int64_t s = 0; s < n; ++s) {
      const int64_t o = c->perm[s];
      const int32_t t = frame_type[o];
      need(t >= 0 && t <= 2, "frames: frame type must be 0, 1 or 2");
      if (t == 0) continue;
      const int32_t zo = zatom[o], xo = xatom[o];
      need(zo >= 0 && zo < n && xo >= 0 && xo < n && zo != o && xo != o && zo != xo,
           "frames: zatom / xatom must be two other sites");
      fr[4 * s] = t;
      fr[4 * s + 1] = c->iperm[zo];
      fr[4 * s + 2] = c->iperm[xo];
      any = true;
      // references that the owned gather can collect: owned site -> owned atom
      if (s < c->n_own) {
        if (fr[4 * s + 1] < c->n_own) ++cnt[fr[4 * s + 1] + 1];
        if (fr[4 * s + 2] < c->n_own) ++cnt[fr[4 * s + 2] + 1];
      }
    }
    for (int64_t a = 0; a < n; ++a) cnt[a + 1] += cnt[a];
    std::vector<int32_t> ref(std::max<int32_t>(cnt[n], 1)), fill(cnt.begin(), cnt.end() - 1);
    for (int64_t s = 0; s < c->n_own; ++s) {
      if (fr[4 * s] == 0) continue;
      for (int role = 0; role < 2; ++role) {
        const int32_t a = fr[4 * s + 1 + role];
        if (a < c->n_own) ref[fill[a]++] = (int32_t)(2 * s + role);
      }
    }
    std::vector<double> ml(12 * n, 0.0);
    for (int64_t s = 0; s < n; ++s) {
      const int64_t o = c->perm[s];
      double* m = &ml[12 * s];
      if (dipole)
        for (int k = 0; k < 3; ++k) m[k] = dipole[3 * o + k];
      if (quadrupole)
        for (int k = 0; k < 6; ++k) m[3 + k] = quadrupole[6 * o + k];
    }
    if (!c->frame) {
      MDG_CUDA_CHECK(cudaMalloc(&c->frame, (size_t)c->n_cap * sizeof(int4)));
      MDG_CUDA_CHECK(cudaMalloc(&c->mploc, 3 * (size_t)c->n_cap * sizeof(double4)));
      MDG_CUDA_CHECK(cudaMalloc(&c->fbuf, 3 * (size_t)c->n_cap * sizeof(double4)));
      MDG_CUDA_CHECK(cudaMalloc(&c->fref_start, ((size_t)c->n_cap + 1) * sizeof(int32_t)));
    }
    if (c->fref) cudaFree(c->fref);
    c->fref = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&c->fref, ref.size() * sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->frame, fr.data(), fr.size() * 4, cudaMemcpyHostToDevice,
                                   c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->mploc, ml.data(), ml.size() * 8, cudaMemcpyHostToDevice,
                                   c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->fref_start, cnt.data(), cnt.size() * 4,
                                   cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->fref, ref.data(), ref.size() * 4, cudaMemcpyHostToDevice,
                                   c->stream));
    c->has_frames = true;  // (frame 0 sites copy their multipoles unrotated)
    c->has_mpoles = true;
    (void)any;
    mdg::rotate_multipoles(c);
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int mdg_multipoles_upload(mdg_ctx* c, const double* dipole, const double* quadrupole) {
  return guard([&] {
    need_system(c);
    set_device(c);
    const int64_t n = c->n;
    std::vector<double> mp(12 * n, 0.0);
    for (int64_t s = 0; s < n; ++s) {
      const int64_t o = c->perm[s];
      double* m = &mp[12 * s];
      if (dipole) {
        m[0] = dipole[3 * o];
        m[1] = dipole[3 * o + 1];
        m[2] = dipole[3 * o + 2];
      }
      if (quadrupole) {
        const double* q = quadrupole + 6 * o;
        m[3] = q[0];  // xx
        m[4] = q[1];  // xy
        m[5] = q[2];  // xz
        m[6] = q[3];  // yy
        m[7] = q[4];  // yz
        m[8] = q[5];  // zz
      }
    }
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->mp, mp.data(), 12 * n * sizeof(double),
                                   cudaMemcpyHostToDevice, c->stream));
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    c->has_mpoles = dipole != nullptr || quadrupole != nullptr;
    c->has_frames = false;  // global-frame multipoles replace any local frames
  });
}

int mdg_nlist_build(mdg_ctx* c, int list_id, double list_cutoff, int sites) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(list_id >= 0 && list_id < MDG_MAX_LISTS, "list id out of range");
    need(sites == MDG_SITES_ATOMIC || sites == MDG_SITES_VDW, "unknown site kind");
    // proj/src/neighbors.cpp:12-17
    need(list_cutoff > 0 && std::isfinite(list_cutoff), "build_cell_grid: cutoff must be positive");
    need(list_cutoff <= 0.5 * std::min(c->lx, std::min(c->ly, c->lz)),
         "build_cell_grid: cutoff exceeds half the smallest box edge");
    mdg::nlist_build(c, list_id, list_cutoff, sites);
  });
}

int mdg_nlist_size(mdg_ctx* c, int list_id, int64_t* half_pairs, int64_t* padded_slots) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    if (half_pairs) *half_pairs = L.half_pairs;
    if (padded_slots) {
      std::vector<int32_t> cnt(c->n), nbr((size_t)c->n * L.cap);
      MDG_CUDA_CHECK(cudaMemcpy(cnt.data(), L.cnt, c->n * 4, cudaMemcpyDeviceToHost));
      MDG_CUDA_CHECK(cudaMemcpy(nbr.data(), L.nbr, nbr.size() * 4, cudaMemcpyDeviceToHost));
      std::vector<int64_t> upper(c->n, 0);
      for (int64_t s = 0; s < c->n; ++s) {
        const int32_t o = c->perm[s];
        const int32_t* row = nbr.data() + (size_t)s * L.cap;
        for (int32_t k = 0; k < cnt[s]; ++k)
          if (c->perm[row[k]] > o) upper[o]++;
      }
      int64_t tot = 0;
      for (int64_t i = 0; i < c->n; ++i) tot += pad_count(upper[i], 16);
      *padded_slots = tot;
    }
  });
}

int mdg_nlist_export(mdg_ctx* c, int list_id, uint32_t* nnvlst, uint32_t* nvloop8,
                     uint32_t* nvloop16, uint64_t* offset, int32_t* indices,
                     int64_t indices_cap) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    const int64_t n = c->n;
    std::vector<int32_t> cnt(n), nbr((size_t)n * L.cap);
    MDG_CUDA_CHECK(cudaMemcpy(cnt.data(), L.cnt, n * 4, cudaMemcpyDeviceToHost));
    MDG_CUDA_CHECK(cudaMemcpy(nbr.data(), L.nbr, nbr.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<std::vector<int32_t>> rows(n);
    for (int64_t s = 0; s < n; ++s) {
      const int32_t o = c->perm[s];
      const int32_t* row = nbr.data() + (size_t)s * L.cap;
      for (int32_t k = 0; k < cnt[s]; ++k) {
        const int32_t jo = c->perm[row[k]];
        if (jo > o) rows[o].push_back(jo);
      }
    }
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i) {
      auto& r = rows[i];
      std::sort(r.begin(), r.end());
      if ((int64_t)r.size() > MDG_MAX_NEIGHBORS)
        throw_error(MDG_CAPACITY, "neighbor table: site " + std::to_string(i) +
                                      " exceeds the per-site neighbor capacity");
      const int64_t k = (int64_t)r.size(), p16 = pad_count(k, 16);
      if (nnvlst) nnvlst[i] = (uint32_t)k;
      if (nvloop8) nvloop8[i] = (uint32_t)pad_count(k, 8);
      if (nvloop16) nvloop16[i] = (uint32_t)p16;
      if (offset) offset[i] = (uint64_t)pos;
      if (indices) {
        need(pos + p16 <= indices_cap, "nlist_export: indices capacity too small");
        const int32_t sentinel = k ? r.back() : 0;
        for (int64_t q = 0; q < p16; ++q) indices[pos + q] = q < k ? r[q] : sentinel;
      }
      pos += p16;
    }
  });
}

int mdg_nlist_import(mdg_ctx* c, int list_id, double list_cutoff, int sites,
                     const uint32_t* nnvlst, const uint64_t* offset, const int32_t* indices) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(list_id >= 0 && list_id < MDG_MAX_LISTS, "list id out of range");
    need(nnvlst && offset && indices, "nlist_import: null array");
    need(list_cutoff > 0, "nlist_import: cutoff must be positive");
    const int64_t n = c->n;
    std::vector<std::vector<int32_t>> rows(n);
    for (int64_t i = 0; i < n; ++i)
      for (uint32_t k = 0; k < nnvlst[i]; ++k) {
        const int32_t j = indices[offset[i] + k];
        need(j >= 0 && j < n && j != i, "nlist_import: neighbour index out of range");
        rows[c->iperm[i]].push_back(c->iperm[j]);
        rows[c->iperm[j]].push_back((int32_t)c->iperm[i]);
      }
    int32_t mx = 0;
    for (auto& r : rows) {
      std::sort(r.begin(), r.end());
      mx = std::max<int32_t>(mx, (int32_t)r.size());
    }
    need(mx <= c->max_pairs, "nlist_import: a site exceeds the context's pair capacity");
    mdg::DevList& L = c->lists[list_id];
    const int32_t cap = std::max<int32_t>(32, (mx + 31) & ~31);
    const size_t need_el = (size_t)n * (size_t)cap;
    if (need_el > L.nbr_elems) {
      if (L.nbr) cudaFree(L.nbr);
      L.nbr = nullptr;
      MDG_CUDA_CHECK(cudaMalloc(&L.nbr, need_el * 4));
      L.nbr_elems = need_el;
    }
    if (!L.cnt) MDG_CUDA_CHECK(cudaMalloc(&L.cnt, (size_t)c->n_cap * 4));
    std::vector<int32_t> ell(need_el, 0), cnt(n);
    int64_t sum = 0;
    for (int64_t s = 0; s < n; ++s) {
      cnt[s] = (int32_t)rows[s].size();
      sum += cnt[s];
      for (size_t k = 0; k < rows[s].size(); ++k)
        ell[(size_t)s * cap + k] = rows[s][k];
    }
    MDG_CUDA_CHECK(cudaMemcpy(L.nbr, ell.data(), need_el * 4, cudaMemcpyHostToDevice));
    MDG_CUDA_CHECK(cudaMemcpy(L.cnt, cnt.data(), n * 4, cudaMemcpyHostToDevice));
    L.cap = cap;
    L.valid = true;
    L.sorted = true;  // rows std::sort-ed above
    L.version = ++c->epoch;
    L.cutoff = list_cutoff;
    L.sites = sites;
    L.max_cnt = mx;
    L.half_pairs = sum / 2;
    mdg::list_snapshot(c, list_id);
  });
}

// ---- kernels -----------------------------------------------------------------

static void nonpolar_call(mdg_ctx* c, int list_id, const mdg::NonpolarArgs& a, double* fx,
                          double* fy, double* fz, double* energy, double* virial9) {
  need_system(c);
  set_device(c);
  mdg::DevList& L = need_list(c, list_id);
  need_kernel_cutoff(L, a.cutoff);
  mdg::run_nonpolar(c, list_id, a);
  vec_out(c, c->force, fx, fy, fz);
  mdg::fetch_results(c);
  if (energy) *energy = a.do_lj ? c->h_results[0] : c->h_results[1];
  if (virial9) sym_virial(c->h_results + 2, virial9);
}

int mdg_lj_forces(mdg_ctx* c, int list_id, double cutoff, int shift, int exclude, double* fx,
                  double* fy, double* fz, double* energy, double* virial9) {
  return guard([&] {
    mdg::NonpolarArgs a{1, 0, shift, exclude, cutoff, 0.0, 1.0};
    nonpolar_call(c, list_id, a, fx, fy, fz, energy, virial9);
  });
}

int mdg_ewald_real_forces(mdg_ctx* c, int list_id, double alpha, double cutoff, double electric,
                          int exclude, double* fx, double* fy, double* fz, double* energy,
                          double* virial9) {
  return guard([&] {
    need(alpha >= 0, "ewald: alpha must be nonnegative");  // kernels_scalar.cpp:58
    mdg::NonpolarArgs a{0, 1, 0, exclude, cutoff, alpha, electric};
    nonpolar_call(c, list_id, a, fx, fy, fz, energy, virial9);
  });
}

int mdg_halgren_forces(mdg_ctx* c, int list_id, double cutoff, double delta, double gamma,
                       int exclude, double* fx, double* fy, double* fz, double* energy,
                       double* virial9) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    mdg::run_halgren(c, list_id, cutoff, delta, gamma, exclude);
    vec_out(c, c->force, fx, fy, fz);
    mdg::fetch_results(c);
    if (energy) *energy = c->h_results[0];
    if (virial9) sym_virial(c->h_results + 2, virial9);
  });
}

int mdg_tmatvec(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                const double* mux, const double* muy, const double* muz, double* ex,
                double* ey, double* ez) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    need(alpha >= 0, "tmatvec: alpha must be nonnegative");
    need(mux && muy && muz, "dipole_field_matvec: dipole array size mismatch");
    need(L.sites == MDG_SITES_ATOMIC, "tmatvec needs a list over atomic sites");
    vec_in(c, mux, muy, muz, c->vin);
    mdg::run_tmatvec(c, list_id, alpha, cutoff, thole_a, c->vin, c->field);
    vec_out(c, c->field, ex, ey, ez);
  });
}

int mdg_perm_field(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                   int exclude, double* ex, double* ey, double* ez) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    need(alpha >= 0, "perm_field: alpha must be nonnegative");
    need(L.sites == MDG_SITES_ATOMIC, "perm_field needs a list over atomic sites");
    mdg::rotate_multipoles(c);
    mdg::run_perm_field(c, list_id, alpha, cutoff, thole_a, exclude, c->field);
    vec_out(c, c->field, ex, ey, ez);
  });
}

int mdg_polar_solve_jacobi(mdg_ctx* c, int list_id, double cutoff, double thole_a, double tol,
                           int64_t max_iter, double* mux, double* muy, double* muz,
                           int64_t* iters, double* last_residual) {
  return guard([&] {
    need_system(c);
    set_device(c);
    // proj/src/polar_scalar.cpp:165-166
    need(tol > 0, "jacobi_polarization_solve: tol must be positive");
    need(max_iter >= 1, "jacobi_polarization_solve: max_iter must be >= 1");
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    mdg::rotate_multipoles(c);
    mdg::run_perm_field(c, list_id, 0.0, cutoff, thole_a, 0, c->eperm);
    double resid = 0;
    try {
      const int64_t it = mdg::run_jacobi(c, list_id, cutoff, thole_a, tol, max_iter, &resid);
      if (iters) *iters = it;
    } catch (const mdg::Error&) {
      if (last_residual) *last_residual = resid;
      if (iters) *iters = max_iter;
      throw;
    }
    if (last_residual) *last_residual = resid;
    vec_out(c, c->mu, mux, muy, muz);
  });
}

int mdg_polar_solve_pcg(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                        int exclude_perm, double tol_debye, int64_t max_iter, double* mux,
                        double* muy, double* muz, int64_t* iters, double* last_rms_debye) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(tol_debye > 0, "pcg: tol must be positive");
    need(max_iter >= 1, "pcg: max_iter must be >= 1");
    need(alpha >= 0, "pcg: alpha must be nonnegative");
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    need(L.sites == MDG_SITES_ATOMIC, "pcg needs a list over atomic sites");
    mdg::rotate_multipoles(c);
    mdg::run_field_tpre(c, list_id, alpha, cutoff, thole_a, exclude_perm);
    if (c->pol_recip.on()) {
      need(alpha > 0, "pcg: reciprocal space needs alpha > 0");
      c->pol_recip.alpha = alpha;
      c->pol_recip.exclude = exclude_perm != 0;
      mdg::pme_field(c, 0, nullptr, c->eperm);
    }
    double rms = 0;
    try {
      const int64_t it = mdg::run_pcg_pre(c, tol_debye, max_iter, &rms);
      if (iters) *iters = it;
    } catch (const mdg::Error&) {
      if (last_rms_debye) *last_rms_debye = rms;
      if (iters) *iters = max_iter;
      throw;
    }
    if (last_rms_debye) *last_rms_debye = rms;
    vec_out(c, c->mu, mux, muy, muz);
  });
}

int mdg_mpole_forces(mdg_ctx* c, int list_id, double alpha, double cutoff, double electric,
                     int exclude, double* fx, double* fy, double* fz, double* tx, double* ty,
                     double* tz, double* energy, double* virial9) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    need(alpha >= 0, "mpole: alpha must be nonnegative");
    need(L.sites == MDG_SITES_ATOMIC, "mpole needs a list over atomic sites");
    mdg::rotate_multipoles(c);
    mdg::run_mpole(c, list_id, alpha, cutoff, electric, exclude, false);
    mdg::frame_torques_to_forces(c);
    vec_out(c, c->force, fx, fy, fz);
    vec_out(c, c->torque, tx, ty, tz);
    mdg::fetch_results(c);
    if (energy) *energy = c->h_results[10];
    if (virial9) std::memcpy(virial9, c->h_results + 11, 9 * sizeof(double));
  });
}

int mdg_polar_forces(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                     double electric, int exclude, const double* mux, const double* muy,
                     const double* muz, double* fx, double* fy, double* fz, double* tx,
                     double* ty, double* tz, double* pair_energy, double* virial9) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, cutoff);
    need(alpha >= 0, "polar_forces: alpha must be nonnegative");
    need(L.sites == MDG_SITES_ATOMIC, "polar_forces needs a list over atomic sites");
    need((mux == nullptr) == (muy == nullptr) && (mux == nullptr) == (muz == nullptr),
         "polar_forces: give all three dipole components or none");
    if (mux) vec_in(c, mux, muy, muz, c->mu);
    mdg::rotate_multipoles(c);
    mdg::run_polar_force(c, list_id, alpha, cutoff, thole_a, electric, exclude, false);
    mdg::frame_torques_to_forces(c);
    vec_out(c, c->force, fx, fy, fz);
    vec_out(c, c->torque, tx, ty, tz);
    mdg::fetch_results(c);
    if (pair_energy) *pair_energy = c->h_results[70];
    if (virial9) std::memcpy(virial9, c->h_results + 71, 9 * sizeof(double));
  });
}

int mdg_ewald_recip_mpole(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order,
                          double electric, int exclude, double* fx, double* fy, double* fz,
                          double* tx, double* ty, double* tz, double* energies3) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(alpha > 0, "ewald_recip_mpole: alpha must be positive");
    need(order >= 5 && order <= 10,
         "ewald_recip_mpole: B-spline order must be 5..10 (third derivatives)");
    need(k1 >= order && k2 >= order && k3 >= order,
         "ewald_recip_mpole: grid smaller than the order");
    need(c->n_own == c->n, "ewald_recip_mpole: single domain only (no distributed FFT)");
    mdg::rotate_multipoles(c);
    MDG_CUDA_CHECK(cudaMemsetAsync(c->force, 0, (size_t)c->n * sizeof(double4), c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(c->torque, 0, (size_t)c->n * sizeof(double4), c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(c->results + 80, 0, 27 * sizeof(double), c->stream));
    mdg::run_pme_mpole(c, alpha, k1, k2, k3, order, electric, exclude != 0);
    vec_out(c, c->force, fx, fy, fz);
    vec_out(c, c->torque, tx, ty, tz);
    mdg::fetch_results(c);
    const double* r = c->h_results;
    if (energies3) {
      const double a2 = alpha * alpha;
      energies3[0] = r[80];
      energies3[1] = -electric * alpha / std::sqrt(M_PI) *
                     (r[104] + 2.0 / 3.0 * a2 * r[105] + 8.0 / 5.0 * a2 * a2 * r[106]);
      energies3[2] = r[88];
    }
  });
}

int mdg_ewald_recip(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order,
                    double electric, int exclude, double* fx, double* fy, double* fz,
                    double* energies3, double* virial9) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(alpha > 0, "ewald_recip: alpha must be positive");
    need(order >= 3 && order <= 10, "ewald_recip: B-spline order must be 3..10");
    need(k1 >= order && k2 >= order && k3 >= order, "ewald_recip: grid smaller than the order");
    need(c->n_own == c->n, "ewald_recip: single domain only (no distributed FFT)");
    MDG_CUDA_CHECK(cudaMemsetAsync(c->force, 0, (size_t)c->n * sizeof(double4), c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(c->results + 80, 0, 18 * sizeof(double), c->stream));
    mdg::run_pme(c, alpha, k1, k2, k3, order, electric, exclude != 0);
    vec_out(c, c->force, fx, fy, fz);
    mdg::fetch_results(c);
    const double* r = c->h_results;
    if (energies3) {
      energies3[0] = r[80];
      energies3[1] = r[87];
      energies3[2] = r[88];
    }
    if (virial9) {
      double w[9];
      sym_virial(r + 81, w);
      for (int k = 0; k < 9; ++k) virial9[k] = w[k] + r[89 + k];
    }
  });
}

// ---- fused steps ---------------------------------------------------------------

// Queue the D2H of the final forces into the registered outputs on the
// current stream (the aux stream while the PCG still runs on the main one).
static void queue_force_output(mdg_ctx* c) {
  if (!c->fout[0]) return;
  mdg::gather_vec_to_caller(c, c->force, c->d_fout);
  for (int a = 0; a < 3; ++a)
    MDG_CUDA_CHECK(cudaMemcpyAsync(c->fout[a], c->d_fout + a * c->n, c->n * sizeof(double),
                                   cudaMemcpyDeviceToHost, c->stream));
  c->fout_seq = g_api_seq.load(std::memory_order_relaxed);
}

int mdg_charmm_step(mdg_ctx* c, int list_id, const mdg_charmm_params* p) {
  return guard([&] {
    need_system(c);
    need(p != nullptr, "null params");
    mdg::DevList& L = need_list(c, list_id);
    need_kernel_cutoff(L, p->cutoff);
    need(L.sites == MDG_SITES_ATOMIC, "charmm step needs a list over atomic sites");
    mdg::NonpolarArgs a{1, 1, p->shift, p->exclude, p->cutoff, p->alpha, p->electric};
    mdg::run_nonpolar(c, list_id, a);
    c->pcg_iters = 0;
    queue_force_output(c);
  });
}

// Halgren + multipoles on the aux stream beside field + PCG (MDG_OVERLAP=0: one stream)
static bool overlap_enabled(mdg_ctx* c) {
  if (!c->overlap) return false;
  if (!c->aux_stream) {
    // the aux chain fills what the critical path (field -> PCG) leaves idle
    int lo = 0, hi = 0;
    MDG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MDG_CUDA_CHECK(cudaStreamCreateWithPriority(&c->aux_stream, cudaStreamNonBlocking, lo));
    for (cudaEvent_t* e : {&c->ev_fork, &c->ev_tpre, &c->ev_join})
      MDG_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  return true;
}

// One domain's AMOEBA step in phases: pre (Halgren + multipoles on the aux
// stream, permanent field + T tensors on the main one), the PCG (one domain,
// or all domains of a group together), post (polarization forces, frames,
// force output). Two independent chains per domain: [aux] Halgren ->
// multipoles (after the pruned rows exist) and [main] permanent field + T ->
// PCG, joined before the polarization forces, which add to the same
// force/torque arrays.
struct AmoebaPhase {
  int terms = 0;
  bool polar = false, late_forces = false, ov = false;
};

static AmoebaPhase amoeba_pre(mdg_ctx* c, int vdw_list, int elec_list, const mdg_amoeba_params* p) {
  need_system(c);
  need(p != nullptr, "null params");
  mdg::DevList& Lv = need_list(c, vdw_list);
  mdg::DevList& Le = need_list(c, elec_list);
  need_kernel_cutoff(Lv, p->vdw_cutoff);
  need_kernel_cutoff(Le, p->elec_cutoff);
  need(Le.sites == MDG_SITES_ATOMIC, "electrostatics need a list over atomic sites");
  AmoebaPhase st;
  st.terms = p->terms ? p->terms : (MDG_TERM_VDW | MDG_TERM_MPOLE | MDG_TERM_POLAR);
  need(!(st.terms & MDG_TERM_POLAR_FORCE) || (st.terms & MDG_TERM_POLAR),
       "amoeba_step: polarization forces need the polarization solve");
  const bool recip = c->pol_recip.on();
  // domains of a group: the reciprocal-space passes run over all domains
  // together (mdg_group_amoeba_step, replicated grid)
  const bool recip_here = recip && c->group == nullptr;
  need(!recip || c->n_own == c->n || c->group != nullptr,
       "amoeba_step: reciprocal space of a domain runs through its group");
  need(!recip || !(st.terms & MDG_TERM_POLAR_FORCE) || (st.terms & MDG_TERM_MPOLE),
       "amoeba_step: reciprocal-space polarization forces come with the multipole term");
  MDG_CUDA_CHECK(cudaMemsetAsync(c->results, 0, (recip ? 107 : 80) * sizeof(double), c->stream));
  c->pol_recip.alpha = p->alpha;
  c->pol_recip.electric = p->electric;
  c->pol_recip.exclude = p->exclude != 0;
  c->recip_in_step = false;
  c->has_polar_force = false;
  mdg::rotate_multipoles(c);  // local frames at the current positions
  // one list for both terms: the two chains would cut / sort the same
  // buffered rows on two unordered streams, so run them on one
  st.ov = vdw_list != elec_list && overlap_enabled(c);
  if (st.ov) {
    MDG_CUDA_CHECK(cudaEventRecord(c->ev_fork, c->stream));
    MDG_CUDA_CHECK(cudaStreamWaitEvent(c->aux_stream, c->ev_fork, 0));
  }
  {
    mdg::AuxScope aux(c, st.ov);
    if (st.terms & MDG_TERM_VDW) {
      mdg::run_halgren(c, vdw_list, p->vdw_cutoff, p->delta, p->gamma, p->exclude);
    } else {
      mdg::zero_vec(c, c->force);
    }
  }
  // With polarization, one pass over the 9 A list prunes it to 7 A, stores
  // the T tensors and computes the permanent field; the multipole kernel
  // then runs on the pruned rows.
  st.polar = (st.terms & MDG_TERM_POLAR) != 0;
  if (st.polar) {
    mdg::run_field_tpre(c, elec_list, p->alpha, p->elec_cutoff, p->thole_a, p->exclude);
    if (recip_here) mdg::pme_field(c, 0, nullptr, c->eperm);  // + reciprocal + self field
    if (st.ov) {
      MDG_CUDA_CHECK(cudaEventRecord(c->ev_tpre, c->stream));
      MDG_CUDA_CHECK(cudaStreamWaitEvent(c->aux_stream, c->ev_tpre, 0));
    }
  }
  // forces are final at the end of the aux chain unless polarization
  // forces or frame torques still add to them
  st.late_forces = (st.polar && (st.terms & MDG_TERM_POLAR_FORCE)) ||
                   (c->has_frames && (st.terms & MDG_TERM_MPOLE)) ||
                   (recip && !recip_here && (st.terms & MDG_TERM_MPOLE));
  {
    mdg::AuxScope aux(c, st.ov);
    if (st.terms & MDG_TERM_MPOLE) {
      if (st.polar) mdg::run_mpole_pruned(c, p->alpha, p->electric, p->exclude, true);
      else mdg::run_mpole(c, elec_list, p->alpha, p->elec_cutoff, p->electric, p->exclude, true);
      if (recip_here) {  // + the multipoles' reciprocal-space sum (own PME state);
        // with polarization forces its forces / torques come from the
        // permanent + induced pass after the solve (amoeba_post)
        const mdg::PolarRecip& R = c->pol_recip;
        const bool combined = st.polar && (st.terms & MDG_TERM_POLAR_FORCE);
        mdg::run_pme_mpole(c, p->alpha, R.k1, R.k2, R.k3, R.order, p->electric, R.exclude,
                           nullptr, !combined);
        c->recip_in_step = true;
      }
    } else {
      mdg::zero_vec(c, c->torque);
    }
    if (!st.late_forces) queue_force_output(c);  // overlaps what is left of the PCG
  }
  c->pcg_iters = -1;  // marks an AMOEBA step for mdg_fetch_energies
  c->pcg_rms = 0;
  return st;
}

// the main stream waits for the aux chain (also when a later stage throws,
// e.g. ConvergenceError from the PCG)
static void amoeba_join(mdg_ctx* c, const AmoebaPhase& st) {
  if (!st.ov) return;
  cudaEventRecord(c->ev_join, c->aux_stream);
  cudaStreamWaitEvent(c->stream, c->ev_join, 0);
}

// post, first part: the real-space polarization forces (and, single
// domain, the combined reciprocal pass); amoeba_post_frames completes
static void amoeba_post_polar(mdg_ctx* c, const AmoebaPhase& st, const mdg_amoeba_params* p) {
  if (st.polar && (st.terms & MDG_TERM_POLAR_FORCE)) {
    mdg::run_polar_force_pruned(c, p->alpha, p->thole_a, p->electric, p->exclude, true);
    if (c->pol_recip.on() && c->group == nullptr && (st.terms & MDG_TERM_MPOLE)) {
      // reciprocal space of multipoles + polarization at fixed dipoles: the
      // forces of the permanent + induced set (E_mpole,rec + E_pol,rec =
      // Q[M + mu], the mu-only self terms being position-independent)
      const mdg::PolarRecip& R = c->pol_recip;
      mdg::run_pme_mpole(c, p->alpha, R.k1, R.k2, R.k3, R.order, p->electric, R.exclude, c->mu,
                         true);
    }
    c->has_polar_force = true;
  }
}

static void amoeba_post_frames(mdg_ctx* c, const AmoebaPhase& st) {
  if ((st.terms & MDG_TERM_MPOLE) || c->has_polar_force) mdg::frame_torques_to_forces(c);
  if (st.late_forces) queue_force_output(c);
}

static void amoeba_post(mdg_ctx* c, const AmoebaPhase& st, const mdg_amoeba_params* p) {
  amoeba_post_polar(c, st, p);
  amoeba_post_frames(c, st);
}

static void amoeba_step_impl(mdg_ctx* c, int vdw_list, int elec_list, const mdg_amoeba_params* p) {
  need(c == nullptr || c->group == nullptr,
       "amoeba_step: this context is a domain of a group (mdg_group_amoeba_step)");
  const AmoebaPhase st = amoeba_pre(c, vdw_list, elec_list, p);
  if (st.polar) {
    double rms = 0;
    try {
      c->pcg_iters = mdg::run_pcg_pre(c, p->tol_debye, p->max_iter, &rms);
    } catch (...) {
      amoeba_join(c, st);
      throw;
    }
    c->pcg_rms = rms;
    mdg::polar_energy(c, p->electric, 40);
  }
  amoeba_join(c, st);
  amoeba_post(c, st, p);
}

int mdg_amoeba_step(mdg_ctx* c, int vdw_list, int elec_list, const mdg_amoeba_params* p) {
  return guard([&] { amoeba_step_impl(c, vdw_list, elec_list, p); });
}

// ---- domain groups (8(e), group.cu): steps and energies over all domains -----

static void energies_of(mdg_ctx* c, double* e4, double* w9);

// reciprocal, self and excluded-pair multipole terms of the last AMOEBA step
// (host results already fetched)
static double recip_energy(const mdg_ctx* c) {
  if (!c->recip_in_step) return 0.0;
  const double* r = c->h_results;
  const double a = c->pol_recip.alpha, a2 = a * a;
  return r[80] + r[88] - c->pol_recip.electric * a / std::sqrt(M_PI) *
                             (r[104] + 2.0 / 3.0 * a2 * r[105] + 8.0 / 5.0 * a2 * a2 * r[106]);
}

int mdg_group_amoeba_step(mdg_group* g, int vdw_list, int elec_list, const mdg_amoeba_params* p) {
  return guard([&] {
    need(g != nullptr, "group: null");
    std::vector<mdg_ctx*> doms = mdg::group_domains(g);
    set_device(doms[0]);
    mdg::group_refresh(g);
    std::vector<AmoebaPhase> st;
    auto join_all = [&] {
      for (size_t k = 0; k < st.size(); ++k) amoeba_join(doms[k], st[k]);
    };
    const bool recip = doms[0]->pol_recip.on();
    mdg::PcgComm* comm = mdg::group_comm(g);
    try {
      for (mdg_ctx* c : doms) st.push_back(amoeba_pre(c, vdw_list, elec_list, p));
      // reciprocal space over all domains (replicated grid): the permanent
      // field before the solve
      if (recip && st[0].polar) mdg::pme_field_multi(doms, comm, 0);
      if (st[0].polar) {
        double rms = 0;
        const int64_t it =
            mdg::run_pcg_multi(doms, mdg::group_comm(g), p->tol_debye, p->max_iter, &rms);
        for (mdg_ctx* c : doms) {
          c->pcg_iters = it;
          c->pcg_rms = rms;
          mdg::polar_energy(c, p->electric, 40);
        }
      }
    } catch (...) {
      join_all();
      throw;
    }
    join_all();
    // the solve leaves the halo dipoles at mu0: refresh them for the forces
    if (st[0].polar && (st[0].terms & MDG_TERM_POLAR_FORCE)) comm->exchange(MDG_VEC_MU);
    for (size_t k = 0; k < st.size(); ++k) amoeba_post_polar(doms[k], st[k], p);
    if (recip && (st[0].terms & MDG_TERM_MPOLE)) {
      // the multipoles' reciprocal sum (energy; forces and torques unless the
      // combined permanent + induced pass below gives them), after the aux
      // chains joined: these passes add to the same force / torque arrays
      const mdg::PolarRecip& R = doms[0]->pol_recip;
      const bool combined = st[0].polar && (st[0].terms & MDG_TERM_POLAR_FORCE);
      mdg::run_pme_mpole_multi(doms, comm, p->alpha, R.k1, R.k2, R.k3, R.order, p->electric,
                               R.exclude, false, !combined);
      if (combined)
        mdg::run_pme_mpole_multi(doms, comm, p->alpha, R.k1, R.k2, R.k3, R.order, p->electric,
                                 R.exclude, true, true);
      for (mdg_ctx* c : doms) c->recip_in_step = true;
    }
    for (size_t k = 0; k < st.size(); ++k) amoeba_post_frames(doms[k], st[k]);
  });
}

int mdg_group_charmm_step(mdg_group* g, int list_id, const mdg_charmm_params* p) {
  return guard([&] {
    need(g != nullptr && p != nullptr, "group: null argument");
    for (mdg_ctx* c : mdg::group_domains(g)) {
      need_system(c);
      mdg::DevList& L = need_list(c, list_id);
      need_kernel_cutoff(L, p->cutoff);
      need(L.sites == MDG_SITES_ATOMIC, "charmm step needs a list over atomic sites");
      mdg::NonpolarArgs a{1, 1, p->shift, p->exclude, p->cutoff, p->alpha, p->electric};
      mdg::run_nonpolar(c, list_id, a);
      c->pcg_iters = 0;
    }
  });
}

int mdg_group_fetch_energies(mdg_group* g, double* energies4, double* virial9,
                             int64_t* pcg_iters, double* pcg_rms) {
  return guard([&] {
    need(g != nullptr, "group: null");
    std::vector<mdg_ctx*> doms = mdg::group_domains(g);
    double v[13] = {0};
    for (mdg_ctx* c : doms) {
      double e[4], w[9];
      energies_of(c, e, w);
      for (int k = 0; k < 4; ++k) v[k] += e[k];
      for (int k = 0; k < 9; ++k) v[4 + k] += w[k];
    }
    mdg::group_sum_host(g, v, 13);
    if (energies4) std::memcpy(energies4, v, 4 * sizeof(double));
    if (virial9) std::memcpy(virial9, v + 4, 9 * sizeof(double));
    if (pcg_iters) *pcg_iters = doms[0]->pcg_iters > 0 ? doms[0]->pcg_iters : 0;
    if (pcg_rms) *pcg_rms = doms[0]->pcg_rms;
  });
}

// ---- MD (8(f)#4) -----------------------------------------------------------------

int mdg_bonded_upload(mdg_ctx* c, int64_t nbonds, const int32_t* bonds, const double* kb,
                      const double* r0, int64_t nangles, const int32_t* angles,
                      const double* ka, const double* theta0) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(nbonds >= 0 && nangles >= 0, "bonded: negative count");
    need(nbonds == 0 || (bonds && kb && r0), "bonded: null bond arrays");
    need(nangles == 0 || (angles && ka && theta0), "bonded: null angle arrays");
    const int64_t n = c->n;
    auto site = [&](int32_t o) {
      need(o >= 0 && o < n, "bonded: site index out of range");
      return c->iperm[o];
    };
    std::vector<int32_t> bij(2 * std::max<int64_t>(nbonds, 1));
    std::vector<double> bp(2 * std::max<int64_t>(nbonds, 1));
    for (int64_t k = 0; k < nbonds; ++k) {
      bij[2 * k] = site(bonds[2 * k]);
      bij[2 * k + 1] = site(bonds[2 * k + 1]);
      bp[2 * k] = kb[k];
      bp[2 * k + 1] = r0[k];
    }
    std::vector<int32_t> aijk(4 * std::max<int64_t>(nangles, 1), 0);
    std::vector<double> ap(2 * std::max<int64_t>(nangles, 1));
    for (int64_t k = 0; k < nangles; ++k) {
      for (int t = 0; t < 3; ++t) aijk[4 * k + t] = site(angles[3 * k + t]);
      ap[2 * k] = ka[k];
      ap[2 * k + 1] = theta0[k];
    }
    for (void** p : {(void**)&c->bond_ij, (void**)&c->bond_par, (void**)&c->angle_ijk,
                     (void**)&c->angle_par}) {
      if (*p) cudaFree(*p);
      *p = nullptr;
    }
    MDG_CUDA_CHECK(cudaMalloc(&c->bond_ij, bij.size() * 4));
    MDG_CUDA_CHECK(cudaMalloc(&c->bond_par, bp.size() * 8));
    MDG_CUDA_CHECK(cudaMalloc(&c->angle_ijk, aijk.size() * 4));
    MDG_CUDA_CHECK(cudaMalloc(&c->angle_par, ap.size() * 8));
    MDG_CUDA_CHECK(cudaMemcpy(c->bond_ij, bij.data(), bij.size() * 4, cudaMemcpyHostToDevice));
    MDG_CUDA_CHECK(cudaMemcpy(c->bond_par, bp.data(), bp.size() * 8, cudaMemcpyHostToDevice));
    MDG_CUDA_CHECK(cudaMemcpy(c->angle_ijk, aijk.data(), aijk.size() * 4, cudaMemcpyHostToDevice));
    MDG_CUDA_CHECK(cudaMemcpy(c->angle_par, ap.data(), ap.size() * 8, cudaMemcpyHostToDevice));
    c->nbonds = nbonds;
    c->nangles = nangles;
  });
}

int mdg_bonded_forces(mdg_ctx* c, double* fx, double* fy, double* fz, double* energies2) {
  return guard([&] {
    need_system(c);
    set_device(c);
    MDG_CUDA_CHECK(cudaMemsetAsync(c->force, 0, (size_t)c->n * sizeof(double4), c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(c->results + 100, 0, 2 * sizeof(double), c->stream));
    mdg::run_bonded(c);
    vec_out(c, c->force, fx, fy, fz);
    mdg::fetch_results(c);
    if (energies2) {
      energies2[0] = c->h_results[100];
      energies2[1] = c->h_results[101];
    }
  });
}

int mdg_velocities_upload(mdg_ctx* c, const double* mass, const double* vx, const double* vy,
                          const double* vz) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(vx && vy && vz, "velocities: null array");
    need(mass || c->has_vel, "velocities: masses required on the first upload");
    const int64_t n = c->n;
    std::vector<double> inv(n);
    if (mass) {
      for (int64_t s = 0; s < n; ++s) {
        const double m = mass[c->perm[s]];
        need(m > 0, "velocities: masses must be positive");
        inv[s] = 1.0 / m;
      }
    }
    if (!c->vel) MDG_CUDA_CHECK(cudaMalloc(&c->vel, (size_t)c->n_cap * sizeof(double4)));
    std::vector<double> w;
    if (!mass) {  // keep the stored 1/m
      std::vector<double4> old(n);
      MDG_CUDA_CHECK(cudaMemcpy(old.data(), c->vel, n * sizeof(double4), cudaMemcpyDeviceToHost));
      for (int64_t s = 0; s < n; ++s) inv[s] = old[s].w;
    }
    std::vector<double4> v(n);
    for (int64_t s = 0; s < n; ++s) {
      const int64_t o = c->perm[s];
      v[s] = make_double4(vx[o], vy[o], vz[o], inv[s]);
    }
    MDG_CUDA_CHECK(cudaMemcpy(c->vel, v.data(), n * sizeof(double4), cudaMemcpyHostToDevice));
    c->has_vel = true;
  });
}

int mdg_velocities_fetch(mdg_ctx* c, double* vx, double* vy, double* vz) {
  return guard([&] {
    need_system(c);
    need(c->has_vel, "velocities: none uploaded");
    vec_out(c, c->vel, vx, vy, vz);
  });
}

int mdg_positions_fetch(mdg_ctx* c, double* x, double* y, double* z) {
  return guard([&] {
    need_system(c);
    vec_out(c, c->pos, x, y, z);
  });
}

int mdg_md_run(mdg_ctx* c, const mdg_md_params* p, const mdg_charmm_params* cp,
               const mdg_amoeba_params* ap, double* ekin, double* epot) {
  return guard([&] {
    need_system(c);
    set_device(c);
    need(p != nullptr, "md: null params");
    need(c->has_vel, "md: upload masses and velocities first");
    need(c->n_own == c->n, "md: single domain only (no migration between domains)");
    need(p->nsteps >= 0 && p->dt_fs > 0 && p->rebuild_every >= 1, "md: bad step parameters");
    need(p->predictor == MDG_PREDICT_NONE || p->predictor == MDG_PREDICT_ASPC,
         "md: unknown dipole predictor");
    need(p->model == 0 ? cp != nullptr : (p->model == 1 && ap != nullptr),
         "md: model 0 needs charmm params, model 1 amoeba params");
    // no per-step force DMA inside the loop (the bonded terms are added after
    // the step's queue point, and the copies would sit on the critical path);
    // a fetch after md_run takes the ordinary path
    struct NoForceOutput {
      mdg_ctx* c;
      double* f[3];
      ~NoForceOutput() {
        for (int a = 0; a < 3; ++a) c->fout[a] = f[a];
        c->fout_seq = 0;
      }
    } nfo{c, {c->fout[0], c->fout[1], c->fout[2]}};
    for (int a = 0; a < 3; ++a) c->fout[a] = nullptr;
    // ASPC dipole prediction for the PCG start (model 1, p->predictor)
    struct AspcScope {
      mdg_ctx* c;
      ~AspcScope() {
        c->aspc_on = false;
        c->aspc_count = 0;
      }
    } aspc{c};
    c->aspc_on = p->model == 1 && p->predictor == MDG_PREDICT_ASPC;
    c->aspc_count = 0;
    c->aspc_head = 0;
    // re-sort the sites by their current cells every MDG_RESORT-th list
    // rebuild (the gathers keep their locality as molecules diffuse: water
    // moves ~1 A per ps, the sort cells are 2 A; 0 = never). The default 20
    // is every 200 fs at the usual 10 fs between rebuilds; a re-sort costs
    // about a third of a config-4 step.
    const int resort = mdg::env_int("MDG_RESORT", 20);
    // a rebuild is due on schedule, or early when the device has flagged a
    // site past 0.6 x its list's tolerable motion (read without a sync: the
    // flag may lag the device by the steps the host has queued ahead)
    // (the warning carries the generation of the lists it is about: a late
    // one about lists already replaced is ignored)
    auto due = [&](int64_t s) {
      return (s + 1) % p->rebuild_every == 0 || *(volatile int32_t*)c->h_warn == c->list_gen;
    };
    auto rebuild = [&] {
      // counted across mdg_md_run calls (a trajectory run in chunks)
      ++c->md_rebuilds;
      if (resort > 0 && c->md_rebuilds % resort == 0) mdg::resort_sites(c);
      mdg::nlist_build(c, p->elec_list, p->elec_list_cutoff, MDG_SITES_ATOMIC);
      if (p->model == 1) mdg::nlist_build(c, p->vdw_list, p->vdw_list_cutoff, MDG_SITES_VDW);
    };
    double e_nb = 0.0;
    auto forces = [&](bool with_bonded) {
      if (p->model == 0) {
        mdg::NonpolarArgs a{1, 1, cp->shift, cp->exclude, cp->cutoff, cp->alpha, cp->electric};
        mdg::run_nonpolar(c, p->elec_list, a);
      } else {
        amoeba_step_impl(c, p->vdw_list, p->elec_list, ap);
      }
      if (with_bonded) {
        MDG_CUDA_CHECK(cudaMemsetAsync(c->results + 100, 0, 2 * sizeof(double), c->stream));
        mdg::run_bonded(c);
      }
    };
    auto potential = [&] {
      const double* r = c->h_results;
      e_nb = (p->model == 0) ? r[0] + r[1] : r[0] + r[10] + r[40] + recip_energy(c);
      return e_nb + (p->bonded ? r[100] + r[101] : 0.0);
    };
    auto report = [&](int64_t s) {
      if (ekin || epot) {
        mdg::run_kinetic(c);
        mdg::fetch_results(c);
        if (ekin) ekin[s] = c->h_results[102];
        if (epot) epot[s] = potential();
      }
    };
    const double dt = p->dt_fs;
    if (p->integrator == MDG_INTEGRATOR_VERLET) {
      rebuild();
      forces(p->bonded);
      for (int64_t s = 0; s < p->nsteps; ++s) {
        mdg::run_kick(c, 0.5 * dt);
        mdg::run_drift(c, dt);
        if (due(s)) rebuild();
        forces(p->bonded);
        mdg::run_kick(c, 0.5 * dt);
        report(s);
      }
    } else {
      // BAOAB-RESPA: c->force holds the outer (nonbonded) forces, c->fbond
      // the inner (bonded) ones
      need(p->integrator == MDG_INTEGRATOR_BAOAB_RESPA, "md: unknown integrator");
      need(p->inner_steps >= 1, "md: BAOAB-RESPA needs inner_steps >= 1");
      need(p->friction_ps >= 0 && p->temperature_k >= 0, "md: negative friction or temperature");
      if (!c->fbond) MDG_CUDA_CHECK(cudaMalloc(&c->fbond, (size_t)c->n_cap * sizeof(double4)));
      const bool bonded = p->bonded && (c->nbonds > 0 || c->nangles > 0);
      auto inner_forces = [&] {
        MDG_CUDA_CHECK(cudaMemsetAsync(c->fbond, 0, (size_t)c->n * sizeof(double4), c->stream));
        MDG_CUDA_CHECK(cudaMemsetAsync(c->results + 100, 0, 2 * sizeof(double), c->stream));
        if (bonded) mdg::run_bonded(c, c->fbond);
      };
      const double h = dt / p->inner_steps;
      const double c1 = std::exp(-p->friction_ps * 1e-3 * h);
      const double kt = 0.0019872041 * p->temperature_k;  // kcal/mol
      const bool langevin = p->friction_ps > 0;
      rebuild();
      forces(false);  // the bonded terms are the inner level
      inner_forces();
      uint64_t counter = 0;
      for (int64_t s = 0; s < p->nsteps; ++s) {
        mdg::run_kick(c, 0.5 * dt);
        for (int k = 0; k < p->inner_steps; ++k) {
          mdg::run_kick(c, 0.5 * h, c->fbond);
          mdg::run_drift(c, 0.5 * h);
          if (langevin) mdg::run_ostep(c, c1, kt, p->seed, counter++);
          mdg::run_drift(c, 0.5 * h);
          inner_forces();
          mdg::run_kick(c, 0.5 * h, c->fbond);
        }
        if (due(s)) {
          rebuild();
          inner_forces();  // a re-sort permuted the sites under c->fbond
        }
        forces(false);  // the bonded terms are the inner level
        mdg::run_kick(c, 0.5 * dt);
        report(s);
      }
    }
    mdg::fetch_results(c);
    mdg::check_lists_fresh(c);  // (rebuild_every too long for this motion)
  });
}

int mdg_md_rebuild_count(mdg_ctx* c, int64_t* count) {
  return guard([&] {
    need_ctx(c);
    need(count != nullptr, "md_rebuild_count: null output");
    *count = c->md_rebuilds;
  });
}

int mdg_resort(mdg_ctx* c) {
  return guard([&] {
    need_system(c);
    set_device(c);
    mdg::resort_sites(c);
  });
}

int mdg_timer_start(mdg_ctx* c) {
  return guard([&] {
    need_ctx(c);
    set_device(c);
    if (!c->timer_a) {
      MDG_CUDA_CHECK(cudaEventCreate(&c->timer_a));
      MDG_CUDA_CHECK(cudaEventCreate(&c->timer_b));
    }
    MDG_CUDA_CHECK(cudaEventRecord(c->timer_a, c->stream));
  });
}

int mdg_timer_stop(mdg_ctx* c, double* ms) {
  return guard([&] {
    need_ctx(c);
    need(c->timer_a != nullptr, "timer not started");
    MDG_CUDA_CHECK(cudaEventRecord(c->timer_b, c->stream));
    MDG_CUDA_CHECK(cudaEventSynchronize(c->timer_b));
    float f = 0;
    MDG_CUDA_CHECK(cudaEventElapsedTime(&f, c->timer_a, c->timer_b));
    if (ms) *ms = f;
  });
}

int mdg_fetch_forces(mdg_ctx* c, double* fx, double* fy, double* fz) {
  return guard([&] {
    need_system(c);
    // the step just before this call already DMA'd into these buffers
    if (c->fout[0] && fx == c->fout[0] && fy == c->fout[1] && fz == c->fout[2] &&
        c->fout_seq + 1 == g_api_seq.load(std::memory_order_relaxed)) {
      MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      if (fx && c->debug_perturb != 0.0) fx[0] += c->debug_perturb;
      return;
    }
    vec_out(c, c->force, fx, fy, fz);
    if (fx && c->debug_perturb != 0.0) fx[0] += c->debug_perturb;
  });
}

int mdg_set_debug_perturb(mdg_ctx* c, double delta) {
  return guard([&] {
    need_ctx(c);
    c->debug_perturb = delta;
  });
}

int mdg_set_force_output(mdg_ctx* c, double* fx, double* fy, double* fz) {
  return guard([&] {
    need_system(c);
    set_device(c);
    MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));  // no DMA into the old buffers in flight
    if (!fx && !fy && !fz) {
      c->fout[0] = c->fout[1] = c->fout[2] = nullptr;
      return;
    }
    need(is_pinned(fx) && is_pinned(fy) && is_pinned(fz),
         "set_force_output: buffers must be page-locked (mdg_host_alloc)");
    if (!c->d_fout) MDG_CUDA_CHECK(cudaMalloc(&c->d_fout, 3 * (size_t)c->n_cap * sizeof(double)));
    c->fout[0] = fx;
    c->fout[1] = fy;
    c->fout[2] = fz;
  });
}

int mdg_fetch_torques(mdg_ctx* c, double* tx, double* ty, double* tz) {
  return guard([&] {
    need_system(c);
    vec_out(c, c->torque, tx, ty, tz);
  });
}

int mdg_fetch_dipoles(mdg_ctx* c, double* mux, double* muy, double* muz) {
  return guard([&] {
    need_system(c);
    vec_out(c, c->mu, mux, muy, muz);
  });
}

int mdg_fetch_perm_field(mdg_ctx* c, double* ex, double* ey, double* ez) {
  return guard([&] {
    need_system(c);
    vec_out(c, c->eperm, ex, ey, ez);
  });
}

// energies: {vdw (lj or halgren), coulomb/multipole, polarization, 0}
static void energies_of(mdg_ctx* c, double* e4, double* w9) {
  mdg::fetch_results(c);
  const double* r = c->h_results;
  double w[9];
  sym_virial(r + 2, w);
  const bool amoeba = c->pcg_iters != 0;
  e4[0] = r[0];
  e4[1] = amoeba ? r[10] : r[1];
  if (amoeba) e4[1] += recip_energy(c);
  e4[2] = amoeba ? r[40] : 0.0;
  e4[3] = 0.0;
  for (int k = 0; k < 9; ++k)
    w9[k] = w[k] + (amoeba ? r[11 + k] : 0.0) + (c->has_polar_force ? r[71 + k] : 0.0);
}

int mdg_fetch_energies(mdg_ctx* c, double* energies4, double* virial9, int64_t* pcg_iters,
                       double* pcg_rms) {
  return guard([&] {
    need_system(c);
    double e[4], w[9];
    energies_of(c, e, w);
    mdg::check_lists_fresh(c);
    e[0] += c->debug_perturb;
    if (energies4) std::memcpy(energies4, e, sizeof e);
    if (virial9) std::memcpy(virial9, w, sizeof w);
    if (pcg_iters) *pcg_iters = c->pcg_iters > 0 ? c->pcg_iters : 0;
    if (pcg_rms) *pcg_rms = c->pcg_rms;
  });
}

int64_t mdg_launch_count(mdg_ctx* c) { return c ? c->launches : 0; }

int mdg_profile_enable(mdg_ctx* c, int enable) {
  return guard([&] {
    need_ctx(c);
    mdg::flush_profile(c);
    c->profile = enable != 0;
  });
}

int mdg_profile_reset(mdg_ctx* c) {
  return guard([&] {
    need_ctx(c);
    mdg::flush_profile(c);
    c->prof.clear();
  });
}

int mdg_profile_report(mdg_ctx* c, char* buf, int64_t buf_len) {
  return guard([&] {
    need_ctx(c);
    need(buf && buf_len > 0, "null buffer");
    mdg::flush_profile(c);
    std::string s;
    char line[256];
    for (auto& kv : c->prof) {
      snprintf(line, sizeof line, "%s %lld %.6f\n", kv.first.c_str(),
               (long long)kv.second.count, kv.second.ms);
      s += line;
    }
    need((int64_t)s.size() < buf_len, "profile report buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
