// group.cu -- spatial domain decomposition runtime.
//
// A group is the set of domain contexts of one decomposed system. Each domain
// owns the molecules whose anchor site lies in its subdomain and holds a halo
// of the neighbouring domains' sites (dd.py builds the plan); every domain
// evaluates the rows of its owned sites, so its owned forces, fields and
// dipoles are complete from owned + halo data.
//
// Inside the PCG solve every iteration refreshes the halo of the search
// direction and sums three CG scalars over all domains; both are device-side
// operations ordered on the domains' stream, so the solve needs no host round
// trip per iteration (PcgComm, polar.cu run_pcg_multi):
//  * LOCAL: several domains in this process on one device. They share one
//    stream; a halo refresh is one kernel per domain that pulls each halo
//    site's vector straight from its owning domain's array (same device), and
//    the scalar sum is one kernel over the domains' result slots in a fixed
//    order. Both are capturable, so the whole multi-domain solve runs as one
//    device-side while graph (and no kernel waits on another domain's: the
//    domains' kernels are serialised on the one stream).
//  * NCCL: one domain per process (rank = GPU). A halo refresh packs the
//    owned sites every peer needs, posts all sends and receives as one NCCL
//    group (ncclSend/ncclRecv over NVLink), and unpacks into the halo; the
//    scalar sum is an in-place ncclAllReduce on the result slots. NCCL is
//    loaded at run time (dlopen libnccl.so.2 -- the copy torch already
//    loaded, else the system one). Iterations are queued in batches ahead of
//    the device (polar.cu).
// Two further operations serve the solve:
//  * interior/halo overlap (exchange_begin / exchange_end): the refresh runs
//    on the group's own highest-priority stream while the domains' stream
//    computes the rows without halo sites (polar.cu pcg_body);
//  * the replicated reciprocal-space grid (grid_sum): LOCAL adds the other
//    domains' grids into the first one (one fixed-order kernel), NCCL
//    all-reduces each rank's grid in place (pme.cu PmeDoms).
// Reference: none (the reference is single-process);
// the model is Tinker-HP's spatial decomposition.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace mdg {

// ---- NCCL, loaded at run time ------------------------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int,
                         ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*ErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name)); };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Reduce, "ncclReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.ErrorString, "ncclGetErrorString");
  });
  if (!api.AllReduce || !api.Send || !api.CommInitRank)
    throw_error(MDG_COMM, "NCCL (libnccl.so.2) not found");
  return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw_error(MDG_COMM, std::string(what) + ": " + nccl().ErrorString(r));
}

// ---- kernels -----------------------------------------------------------------
// halo site dst[k] of a domain <- the same site's entry in its owning domain
// (src[k] = (domain, sorted index)); POS keeps the w word (group/type bits)
__global__ void k_halo_pull(int64_t nh, const int32_t* __restrict__ dst,
                            const int2* __restrict__ src, double4* const* __restrict__ vecs,
                            double4* __restrict__ out, const double* __restrict__ res,
                            int skip_converged) {
  if (skip_converged && res[27] != 0.0) return;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nh) return;
  const int2 s = src[k];
  const double4 v = vecs[s.x][s.y];
  double4* o = out + dst[k];
  o->x = v.x;
  o->y = v.y;
  o->z = v.z;
}

// res_d[slot + v] <- sum over domains d (fixed order), for every domain
__global__ void k_group_sum(double* const* __restrict__ res, int ndom, int slot, int nv) {
  const int v = threadIdx.x;
  if (v >= nv) return;
  if (res[0][27] != 0.0 && slot != 21) return;  // converged (speculative iteration)
  double s = 0.0;
  for (int d = 0; d < ndom; ++d) s += res[d][slot + v];
  for (int d = 0; d < ndom; ++d) res[d][slot + v] = s;
}

__global__ void k_pack3(int64_t n, const int32_t* __restrict__ idx, const double4* __restrict__ v,
                        double* __restrict__ out, const double* __restrict__ res, int skip) {
  if (skip && res[27] != 0.0) return;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double4 a = v[idx[k]];
  out[3 * k] = a.x;
  out[3 * k + 1] = a.y;
  out[3 * k + 2] = a.z;
}

__global__ void k_unpack3(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ in,
                          double4* __restrict__ v, const double* __restrict__ res, int skip) {
  if (skip && res[27] != 0.0) return;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double4* a = v + idx[k];
  a->x = in[3 * k];
  a->y = in[3 * k + 1];
  a->z = in[3 * k + 2];
}

// replicated-grid reciprocal space on one device: g[0] += g[1] + ... (a
// fixed order)
constexpr int kMaxGridDoms = 16;
struct GridPtrs {
  double* g[kMaxGridDoms];
};

__global__ void k_grid_sum(size_t count, GridPtrs p, int nd) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = p.g[0][i];
    for (int d = 1; d < nd; ++d) s += p.g[d][i];
    p.g[0][i] = s;
  }
}

// slab-decomposed reciprocal space on one device: element i of the grid, in
// part p's planes [off[p], off[p+1]), <- the sum over the domains' grids (the
// same fixed order as k_grid_sum), written into part p's own grid
struct SlabOff {
  int64_t o[kMaxGridDoms + 1];
};

__global__ void k_slab_reduce(size_t count, GridPtrs p, int nd, SlabOff off) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    int part = 0;
    while (part + 1 < nd && (int64_t)i >= off.o[part + 1]) ++part;
    double s = p.g[0][i];
    for (int d = 1; d < nd; ++d) s += p.g[d][i];
    p.g[part][i] = s;
  }
}

// max |minimum image (pos - ref)|^2 over the owned sites, as ordered bits
__global__ void k_max_disp2(int64_t n, Box b, const double4* __restrict__ pos,
                            const double4* __restrict__ ref, unsigned long long* __restrict__ out) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (s < n) {
    const double4 p = pos[s], r = ref[s];
    double dx, dy, dz;
    d2 = min_image(b, p.x, p.y, p.z, r.x, r.y, r.z, dx, dy, dz);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d2 = fmax(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(d2));
}

void refresh_vsites(mdg_ctx* c);  // core.cu: vdW sites after new halo positions

}  // namespace mdg

using namespace mdg;

struct mdg_group : PcgComm {
  int backend = MDG_GROUP_LOCAL;
  int rank = 0, size = 1;
  int64_t nglob = 0;
  uintptr_t gen = 1;
  std::vector<mdg_ctx*> dom;
  std::vector<cudaStream_t> own_stream;  // LOCAL: each context's own stream, restored at destroy
  // LOCAL halo: per domain, halo sites (sorted index) and their sources
  struct LocalHalo {
    int64_t n = 0;
    int32_t* dst = nullptr;
    int2* src = nullptr;
  };
  std::vector<LocalHalo> lh;
  double4** d_vecs = nullptr;  // [6][ndom] vector base pointers
  double** d_res = nullptr;    // [ndom] result slots
  std::vector<double4*> h_vecs;  // host copies of the two tables
  std::vector<double*> h_res;
  // NCCL
  ncclComm_t comm = nullptr;
  struct Peer {
    int rank;
    int64_t nsend, nrecv, soff, roff;
  };
  std::vector<Peer> peers;
  int32_t* d_send = nullptr;  // sorted indices, per peer back to back
  int32_t* d_recv = nullptr;
  double* d_sbuf = nullptr;
  double* d_rbuf = nullptr;
  int64_t nsend = 0, nrecv = 0;
  double* d_sum = nullptr;  // energy / virial all-reduce buffer
  std::vector<double4*> ref;  // per domain: positions when the plan was made
  unsigned long long* d_disp = nullptr;
  // interior/halo overlap: the halo refresh of the PCG direction runs on
  // its own (highest-priority) stream while the interior rows are computed
  bool ov = false;
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;

  cudaStream_t stream() const { return dom[0]->stream; }

  void exchange(int vec_id) override { exchange_vec(vec_id, vec_id == MDG_VEC_P, stream()); }

  void grid_sum(double* const* grids, int n, size_t count) override {
    if (backend == MDG_GROUP_LOCAL) {
      if (n <= 1) return;
      if (n > kMaxGridDoms) throw_error(MDG_CONTRACT, "group: too many domains for the grid sum");
      GridPtrs p{};
      for (int d = 0; d < n; ++d) p.g[d] = grids[d];
      dom[0]->launches++;
      k_grid_sum<<<148 * 8, 256, 0, stream()>>>(count, p, n);
    } else if (size > 1) {
      nccl_check(nccl().AllReduce(grids[0], grids[0], count, ncclDouble, ncclSum, comm, stream()),
                 "ncclAllReduce (grid)");
    }
  }
  bool grid_shared() const override { return backend == MDG_GROUP_LOCAL; }

  // slab-decomposed reciprocal space. Default: on for NCCL at world size
  // > 1 (each rank transforms 1/P of the grid instead of all of it), off
  // for LOCAL (one device: the parts' transforms serialise on one stream,
  // the replicated grid transforms once); MDG_PME_SLAB=1 / 0 forces it.
  // LOCAL: the domains are the parts, the transposes are device copies on
  // the one stream. NCCL: the ranks are the parts; grouped ncclReduce /
  // ncclSend+ncclRecv / ncclBroadcast per part.
  int slab_parts() const override {
    const char* e = getenv("MDG_PME_SLAB");
    const bool on = e ? atoi(e) != 0 : (backend != MDG_GROUP_LOCAL && size > 1);
    if (!on) return 0;
    const int P = backend == MDG_GROUP_LOCAL ? (int)dom.size() : size;
    if (P > kMaxGridDoms) throw_error(MDG_CONTRACT, "group: too many parts for the slab FFT");
    return P;
  }
  int slab_part(int d) const override { return backend == MDG_GROUP_LOCAL ? d : rank; }
  void slab_reduce(double* const* grids, int n, const int64_t* off) override {
    const int P = slab_parts();
    if (backend == MDG_GROUP_LOCAL) {
      if (n <= 1) return;
      GridPtrs p{};
      SlabOff o{};
      for (int d = 0; d < n; ++d) p.g[d] = grids[d];
      for (int q = 0; q <= P; ++q) o.o[q] = off[q];
      dom[0]->launches++;
      k_slab_reduce<<<148 * 8, 256, 0, stream()>>>((size_t)off[P], p, n, o);
    } else {
      nccl_check(nccl().GroupStart(), "ncclGroupStart");
      for (int q = 0; q < P; ++q)
        nccl_check(nccl().Reduce(grids[0] + off[q], grids[0] + off[q], off[q + 1] - off[q],
                                 ncclDouble, ncclSum, q, comm, stream()),
                   "ncclReduce (slab)");
      nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    }
  }
  void slab_alltoall(cufftDoubleComplex* const* src, cufftDoubleComplex* const* dst, int n,
                     const int64_t* soff, const int64_t* doff, const int64_t* cnt) override {
    const int P = slab_parts();
    const size_t z = sizeof(cufftDoubleComplex);
    if (backend == MDG_GROUP_LOCAL) {
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < P; ++q)
          if (cnt[p * P + q])
            MDG_CUDA_CHECK(cudaMemcpyAsync(dst[q] + doff[q * P + p], src[p] + soff[p * P + q],
                                           cnt[p * P + q] * z, cudaMemcpyDeviceToDevice,
                                           stream()));
    } else {
      const int r = rank;
      nccl_check(nccl().GroupStart(), "ncclGroupStart");
      for (int q = 0; q < P; ++q) {
        if (cnt[r * P + q])
          nccl_check(nccl().Send(src[0] + soff[r * P + q], 2 * cnt[r * P + q], ncclDouble, q,
                                 comm, stream()),
                     "ncclSend (slab)");
        if (cnt[q * P + r])
          nccl_check(nccl().Recv(dst[0] + doff[r * P + q], 2 * cnt[q * P + r], ncclDouble, q,
                                 comm, stream()),
                     "ncclRecv (slab)");
      }
      nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    }
  }
  void slab_allgather(double* const* grids, int n, const int64_t* off) override {
    const int P = slab_parts();
    if (backend == MDG_GROUP_LOCAL) {
      for (int q = 1; q < n; ++q)
        MDG_CUDA_CHECK(cudaMemcpyAsync(grids[0] + off[q], grids[q] + off[q],
                                       (off[q + 1] - off[q]) * sizeof(double),
                                       cudaMemcpyDeviceToDevice, stream()));
    } else {
      nccl_check(nccl().GroupStart(), "ncclGroupStart");
      for (int q = 0; q < P; ++q)
        nccl_check(nccl().Broadcast(grids[0] + off[q], grids[0] + off[q], off[q + 1] - off[q],
                                    ncclDouble, q, comm, stream()),
                   "ncclBroadcast (slab)");
      nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    }
  }
  bool recip_root(int d) const override {
    return backend == MDG_GROUP_LOCAL ? d == 0 : rank == 0;
  }

  bool overlap() const override {
    if (!ov) return false;
    if (backend == MDG_GROUP_NCCL) return size > 1;
    for (const LocalHalo& h : lh)
      if (h.n) return true;
    return false;
  }

  void exchange_begin(int vec_id) override {
    MDG_CUDA_CHECK(cudaEventRecord(ev_ready, stream()));
    MDG_CUDA_CHECK(cudaStreamWaitEvent(cstream, ev_ready, 0));
    exchange_vec(vec_id, vec_id == MDG_VEC_P, cstream);
    MDG_CUDA_CHECK(cudaEventRecord(ev_done, cstream));
  }

  void exchange_end() override { MDG_CUDA_CHECK(cudaStreamWaitEvent(stream(), ev_done, 0)); }

  // the refresh ops, queued on stream s (the domains' stream, or the
  // communication stream between exchange_begin / exchange_end)
  void exchange_vec(int vec_id, bool skip_converged, cudaStream_t s) {
    if (size == 1 && backend == MDG_GROUP_NCCL) return;
    if (backend == MDG_GROUP_LOCAL) {
      const int nd = (int)dom.size();
      for (int d = 0; d < nd; ++d) {
        mdg_ctx* c = dom[d];
        if (lh[d].n == 0) continue;
        c->launches++;
        k_halo_pull<<<grid_for(lh[d].n, 256), 256, 0, s>>>(
            lh[d].n, lh[d].dst, lh[d].src, d_vecs + (size_t)vec_id * nd, vec_by_id(c, vec_id),
            c->results, skip_converged ? 1 : 0);
      }
    } else {
      mdg_ctx* c = dom[0];
      const NcclApi& N = nccl();
      double4* v = vec_by_id(c, vec_id);
      if (nsend) {
        c->launches++;
        k_pack3<<<grid_for(nsend, 256), 256, 0, s>>>(nsend, d_send, v, d_sbuf, c->results,
                                                     skip_converged ? 1 : 0);
      }
      nccl_check(N.GroupStart(), "ncclGroupStart");
      for (const Peer& p : peers) {
        if (p.nrecv)
          nccl_check(N.Recv(d_rbuf + 3 * p.roff, 3 * p.nrecv, ncclDouble, p.rank, comm, s),
                     "ncclRecv");
        if (p.nsend)
          nccl_check(N.Send(d_sbuf + 3 * p.soff, 3 * p.nsend, ncclDouble, p.rank, comm, s),
                     "ncclSend");
      }
      nccl_check(N.GroupEnd(), "ncclGroupEnd");
      if (nrecv) {
        c->launches++;
        k_unpack3<<<grid_for(nrecv, 256), 256, 0, s>>>(nrecv, d_recv, d_rbuf, v, c->results,
                                                       skip_converged ? 1 : 0);
      }
    }
    if (vec_id == MDG_VEC_POS)
      for (mdg_ctx* c : dom) refresh_vsites(c);
  }

  void init_overlap(bool on) {
    ov = on;
    if (cstream) return;
    int lo = 0, hi = 0;
    MDG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MDG_CUDA_CHECK(cudaStreamCreateWithPriority(&cstream, cudaStreamNonBlocking, hi));
    MDG_CUDA_CHECK(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
    MDG_CUDA_CHECK(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
  }

  void allreduce(int slot, int nv) override {
    if (backend == MDG_GROUP_LOCAL) {
      if (dom.size() == 1) return;
      dom[0]->launches++;
      k_group_sum<<<1, 32, 0, stream()>>>(d_res, (int)dom.size(), slot, nv);
    } else if (size > 1) {
      mdg_ctx* c = dom[0];
      nccl_check(nccl().AllReduce(c->results + slot, c->results + slot, nv, ncclDouble, ncclSum,
                                  comm, c->stream),
                 "ncclAllReduce");
    }
  }

  bool capturable() const override { return backend == MDG_GROUP_LOCAL; }
  int64_t n_global() const override { return nglob; }
  uintptr_t generation() const override { return gen; }
};

namespace {

template <class F>
int gguard(F&& f) {
  try {
    f();
    return MDG_OK;
  } catch (const mdg::Error& e) {
    mdg::set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    mdg::set_error(e.what());
    return MDG_CUDA;
  }
}

void gneed(bool ok, const char* msg) {
  if (!ok) throw_error(MDG_CONTRACT, msg);
}

void refresh_tables(mdg_group* g) {
  const int nd = (int)g->dom.size();
  std::vector<double4*> vecs((size_t)6 * nd);
  std::vector<double*> res(nd);
  for (int v = 0; v < 6; ++v)
    for (int d = 0; d < nd; ++d) vecs[(size_t)v * nd + d] = vec_by_id(g->dom[d], v);
  for (int d = 0; d < nd; ++d) res[d] = g->dom[d]->results;
  // unchanged tables: no copy (a synchronous copy per exchange would stall
  // the host's run-ahead)
  if (g->d_vecs && vecs == g->h_vecs && res == g->h_res) return;
  if (!g->d_vecs) MDG_CUDA_CHECK(cudaMalloc(&g->d_vecs, vecs.size() * sizeof(double4*)));
  if (!g->d_res) MDG_CUDA_CHECK(cudaMalloc(&g->d_res, res.size() * sizeof(double*)));
  MDG_CUDA_CHECK(cudaMemcpy(g->d_vecs, vecs.data(), vecs.size() * sizeof(double4*),
                            cudaMemcpyHostToDevice));
  MDG_CUDA_CHECK(cudaMemcpy(g->d_res, res.data(), res.size() * sizeof(double*),
                            cudaMemcpyHostToDevice));
  g->h_vecs = vecs;
  g->h_res = res;
}

}  // namespace

extern "C" {

int mdg_nccl_unique_id(void* id128) {
  return gguard([&] {
    gneed(id128 != nullptr, "nccl_unique_id: null buffer");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof id);
  });
}

int mdg_group_create_local(mdg_group** out, int n, mdg_ctx** ctxs, int64_t n_global) {
  return gguard([&] {
    gneed(out && n >= 1 && ctxs, "group: bad arguments");
    for (int d = 0; d < n; ++d) {
      gneed(ctxs[d] && ctxs[d]->has_system, "group: every domain needs a system");
      gneed(ctxs[d]->device == ctxs[0]->device, "group: LOCAL domains share one device");
      gneed(ctxs[d]->group == nullptr, "group: context already in a group");
    }
    auto* g = new mdg_group();
    g->backend = MDG_GROUP_LOCAL;
    g->size = n;
    g->nglob = n_global;
    for (int d = 0; d < n; ++d) {
      g->dom.push_back(ctxs[d]);
      g->own_stream.push_back(ctxs[d]->stream);
      ctxs[d]->stream = ctxs[0]->stream;  // one stream: domains ordered, no cross-waits
      ctxs[d]->group = g;
    }
    g->lh.resize(n);
    MDG_CUDA_CHECK(cudaSetDevice(ctxs[0]->device));
    refresh_tables(g);
    // in one process the halo pull is a small kernel beside the mat-vec:
    // the split costs more than it hides (MDG_DD_OVERLAP=1 turns it on)
    g->init_overlap(env_int("MDG_DD_OVERLAP", 0) != 0);
    *out = g;
  });
}

int mdg_group_create_nccl(mdg_group** out, mdg_ctx* ctx, int rank, int size, const void* id128,
                          int64_t n_global) {
  return gguard([&] {
    gneed(out && ctx && ctx->has_system && id128, "group: bad arguments");
    gneed(size >= 1 && rank >= 0 && rank < size, "group: bad rank / size");
    gneed(ctx->group == nullptr, "group: context already in a group");
    MDG_CUDA_CHECK(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t comm = nullptr;
    nccl_check(nccl().CommInitRank(&comm, size, id, rank), "ncclCommInitRank");
    auto* g = new mdg_group();
    g->backend = MDG_GROUP_NCCL;
    g->rank = rank;
    g->size = size;
    g->nglob = n_global;
    g->comm = comm;
    g->dom.push_back(ctx);
    g->own_stream.push_back(ctx->stream);
    g->lh.resize(1);
    ctx->group = g;
    MDG_CUDA_CHECK(cudaMalloc(&g->d_sum, 32 * sizeof(double)));
    // between GPUs the send/receive latency is worth hiding (MDG_DD_OVERLAP=0 off)
    g->init_overlap(env_int("MDG_DD_OVERLAP", 1) != 0);
    *out = g;
  });
}

int mdg_group_destroy(mdg_group* g) {
  return gguard([&] {
    if (!g) return;
    cudaStreamSynchronize(g->stream());
    mdg::pcg_graph_forget(g);
    for (size_t d = 0; d < g->dom.size(); ++d) {
      g->dom[d]->stream = g->own_stream[d];
      g->dom[d]->group = nullptr;
    }
    for (auto& h : g->lh) {
      cudaFree(h.dst);
      cudaFree(h.src);
    }
    for (void* p : {(void*)g->d_vecs, (void*)g->d_res, (void*)g->d_send, (void*)g->d_recv,
                    (void*)g->d_sbuf, (void*)g->d_rbuf, (void*)g->d_sum, (void*)g->d_disp})
      if (p) cudaFree(p);
    for (double4* r : g->ref) cudaFree(r);
    if (g->cstream) cudaStreamSynchronize(g->cstream);
    if (g->ev_ready) cudaEventDestroy(g->ev_ready);
    if (g->ev_done) cudaEventDestroy(g->ev_done);
    if (g->cstream) cudaStreamDestroy(g->cstream);
    if (g->comm) nccl().CommDestroy(g->comm);
    delete g;
  });
}

int mdg_group_set_overlap(mdg_group* g, int on) {
  return gguard([&] {
    gneed(g != nullptr, "group: null");
    MDG_CUDA_CHECK(cudaSetDevice(g->dom[0]->device));
    g->init_overlap(on != 0);
  });
}

int mdg_group_set_halo_local(mdg_group* g, int domain, int64_t n_halo, const int32_t* halo_site,
                             const int32_t* src_domain, const int32_t* src_site) {
  return gguard([&] {
    gneed(g && g->backend == MDG_GROUP_LOCAL, "set_halo_local: not a LOCAL group");
    gneed(domain >= 0 && domain < (int)g->dom.size(), "set_halo_local: bad domain");
    mdg_ctx* c = g->dom[domain];
    gneed(n_halo >= 0 && n_halo <= c->n - c->n_own, "set_halo_local: more halo sites than the domain has");
    std::vector<int32_t> dst(std::max<int64_t>(n_halo, 1));
    std::vector<int2> src(std::max<int64_t>(n_halo, 1));
    for (int64_t k = 0; k < n_halo; ++k) {
      gneed(halo_site[k] >= 0 && halo_site[k] < c->n, "set_halo_local: halo site out of range");
      const int32_t s = c->iperm[halo_site[k]];
      gneed(s >= c->n_own, "set_halo_local: an owned site listed as halo");
      const int q = src_domain[k];
      gneed(q >= 0 && q < (int)g->dom.size() && q != domain, "set_halo_local: bad source domain");
      mdg_ctx* cq = g->dom[q];
      gneed(src_site[k] >= 0 && src_site[k] < cq->n, "set_halo_local: source site out of range");
      const int32_t t = cq->iperm[src_site[k]];
      gneed(t < cq->n_own, "set_halo_local: source site is not owned by the source domain");
      dst[k] = s;
      src[k] = make_int2(q, t);
    }
    auto& h = g->lh[domain];
    cudaFree(h.dst);
    cudaFree(h.src);
    h.dst = nullptr;
    h.src = nullptr;
    MDG_CUDA_CHECK(cudaMalloc(&h.dst, dst.size() * sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMalloc(&h.src, src.size() * sizeof(int2)));
    MDG_CUDA_CHECK(cudaMemcpy(h.dst, dst.data(), dst.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    MDG_CUDA_CHECK(cudaMemcpy(h.src, src.data(), src.size() * sizeof(int2), cudaMemcpyHostToDevice));
    h.n = n_halo;
    refresh_tables(g);  // vectors may have been reallocated by a new upload
    g->gen++;
  });
}

int mdg_group_set_halo_nccl(mdg_group* g, int npeers, const int32_t* peers,
                            const int64_t* send_counts, const int32_t* send_sites,
                            const int64_t* recv_counts, const int32_t* recv_sites) {
  return gguard([&] {
    gneed(g && g->backend == MDG_GROUP_NCCL, "set_halo_nccl: not an NCCL group");
    gneed(npeers >= 0 && (npeers == 0 || (peers && send_counts && recv_counts)),
          "set_halo_nccl: bad arguments");
    mdg_ctx* c = g->dom[0];
    g->peers.clear();
    int64_t ns = 0, nr = 0;
    for (int p = 0; p < npeers; ++p) {
      gneed(peers[p] >= 0 && peers[p] < g->size && peers[p] != g->rank, "set_halo_nccl: bad peer");
      gneed(send_counts[p] >= 0 && recv_counts[p] >= 0, "set_halo_nccl: negative count");
      g->peers.push_back({peers[p], send_counts[p], recv_counts[p], ns, nr});
      ns += send_counts[p];
      nr += recv_counts[p];
    }
    std::vector<int32_t> s(std::max<int64_t>(ns, 1)), r(std::max<int64_t>(nr, 1));
    for (int64_t k = 0; k < ns; ++k) {
      gneed(send_sites[k] >= 0 && send_sites[k] < c->n, "set_halo_nccl: send site out of range");
      s[k] = c->iperm[send_sites[k]];
      gneed(s[k] < c->n_own, "set_halo_nccl: send site is not owned");
    }
    for (int64_t k = 0; k < nr; ++k) {
      gneed(recv_sites[k] >= 0 && recv_sites[k] < c->n, "set_halo_nccl: recv site out of range");
      r[k] = c->iperm[recv_sites[k]];
      gneed(r[k] >= c->n_own, "set_halo_nccl: recv site is owned");
    }
    for (void** p : {(void**)&g->d_send, (void**)&g->d_recv, (void**)&g->d_sbuf, (void**)&g->d_rbuf}) {
      cudaFree(*p);
      *p = nullptr;
    }
    MDG_CUDA_CHECK(cudaMalloc(&g->d_send, s.size() * sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMalloc(&g->d_recv, r.size() * sizeof(int32_t)));
    MDG_CUDA_CHECK(cudaMalloc(&g->d_sbuf, 3 * s.size() * sizeof(double)));
    MDG_CUDA_CHECK(cudaMalloc(&g->d_rbuf, 3 * r.size() * sizeof(double)));
    MDG_CUDA_CHECK(cudaMemcpy(g->d_send, s.data(), s.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    MDG_CUDA_CHECK(cudaMemcpy(g->d_recv, r.data(), r.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    g->nsend = ns;
    g->nrecv = nr;
    g->gen++;
  });
}

int mdg_group_exchange(mdg_group* g, int vec_id) {
  return gguard([&] {
    gneed(g != nullptr, "group: null");
    gneed(vec_id >= 0 && vec_id < 6, "group_exchange: unknown vector id");
    MDG_CUDA_CHECK(cudaSetDevice(g->dom[0]->device));
    if (g->backend == MDG_GROUP_LOCAL) refresh_tables(g);
    // stream-ordered: the next step (or a fetch) sees the refreshed halo
    g->exchange_vec(vec_id, false, g->stream());
  });
}

int mdg_group_set_reference(mdg_group* g) {
  return gguard([&] {
    gneed(g != nullptr, "group: null");
    MDG_CUDA_CHECK(cudaSetDevice(g->dom[0]->device));
    g->ref.resize(g->dom.size(), nullptr);
    for (size_t d = 0; d < g->dom.size(); ++d) {
      mdg_ctx* c = g->dom[d];
      if (!g->ref[d]) MDG_CUDA_CHECK(cudaMalloc(&g->ref[d], (size_t)c->n_cap * sizeof(double4)));
      MDG_CUDA_CHECK(cudaMemcpyAsync(g->ref[d], c->pos, (size_t)c->n_own * sizeof(double4),
                                     cudaMemcpyDeviceToDevice, c->stream));
    }
    MDG_CUDA_CHECK(cudaStreamSynchronize(g->stream()));
  });
}

int mdg_group_max_displacement(mdg_group* g, double* out) {
  return gguard([&] {
    gneed(g != nullptr && out != nullptr, "group: null");
    gneed(g->ref.size() == g->dom.size(), "max_displacement: no reference (mdg_group_set_reference)");
    MDG_CUDA_CHECK(cudaSetDevice(g->dom[0]->device));
    if (!g->d_disp) MDG_CUDA_CHECK(cudaMalloc(&g->d_disp, sizeof(unsigned long long)));
    cudaStream_t s = g->stream();
    MDG_CUDA_CHECK(cudaMemsetAsync(g->d_disp, 0, sizeof(unsigned long long), s));
    for (size_t d = 0; d < g->dom.size(); ++d) {
      mdg_ctx* c = g->dom[d];
      c->launches++;
      k_max_disp2<<<grid_for(c->n_own, 256), 256, 0, c->stream>>>(
          c->n_own, make_box(c->lx, c->ly, c->lz), c->pos, g->ref[d], g->d_disp);
    }
    double d2 = 0.0;
    if (g->backend == MDG_GROUP_NCCL && g->size > 1)
      nccl_check(nccl().AllReduce(g->d_disp, g->d_disp, 1, ncclUint64, ncclMax, g->comm, s),
                 "ncclAllReduce");
    unsigned long long bits = 0;
    MDG_CUDA_CHECK(cudaMemcpyAsync(&bits, g->d_disp, sizeof bits, cudaMemcpyDeviceToHost, s));
    MDG_CUDA_CHECK(cudaStreamSynchronize(s));
    std::memcpy(&d2, &bits, sizeof d2);
    *out = std::sqrt(d2);
  });
}

int mdg_group_allreduce_results(mdg_group* g, int slot, int nv) {
  return gguard([&] {
    gneed(g && slot >= 0 && nv >= 1 && slot + nv <= kResultSlots && nv <= 32,
          "group_allreduce: bad slots");
    g->allreduce(slot, nv);
  });
}

}  // extern "C"

// the group's PcgComm for the step / solve entry points in abi.cpp
namespace mdg {
PcgComm* group_comm(mdg_group* g) { return g; }
std::vector<mdg_ctx*> group_domains(mdg_group* g) { return g->dom; }
bool group_is_nccl(mdg_group* g) { return g->backend == MDG_GROUP_NCCL; }
bool group_overlap(const mdg_ctx* c) { return c->group && c->group->ov; }
void group_refresh(mdg_group* g) {
  if (g->backend == MDG_GROUP_LOCAL) refresh_tables(g);
}
// energies4 + virial9 summed over the ranks of an NCCL group (in place)
void group_sum_host(mdg_group* g, double* v, int nv) {
  if (g->backend != MDG_GROUP_NCCL || g->size == 1) return;
  mdg_ctx* c = g->dom[0];
  MDG_CUDA_CHECK(cudaMemcpyAsync(g->d_sum, v, nv * sizeof(double), cudaMemcpyHostToDevice,
                                 c->stream));
  nccl_check(nccl().AllReduce(g->d_sum, g->d_sum, nv, ncclDouble, ncclSum, g->comm, c->stream),
             "ncclAllReduce");
  MDG_CUDA_CHECK(cudaMemcpyAsync(v, g->d_sum, nv * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
}
}  // namespace mdg
