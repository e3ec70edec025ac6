// resort.cu -- spatial re-sort of the resident sites on the device
// (VERDICT r1 next 7). The site order is a Morton order over ~2 A cells of
// the positions at upload; as sites move, consecutive sites drift apart and
// the pair kernels' gathers lose their cache locality. At a list rebuild
// (mdg_md_run) or on request (mdg_resort) the sites are re-keyed from their
// current positions (the host spatial_sort's keys), radix-sorted (CUB, stable:
// ties keep their previous order) and every per-site array is permuted on the
// device; arrays holding site indices (Halgren parents and children, frame
// atoms, exclusion partners, frame-force references, bonds, angles, the
// caller <-> sorted maps) are remapped. Lists, buffered rows and pruned rows
// are invalidated (the caller rebuilds them next). Single domain only (a
// domain's halo maps are in sorted indices).
#include <cub/cub.cuh>

#include "common.cuh"

namespace mdg {

__device__ __forceinline__ uint64_t spread3_dev(uint64_t v) {
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

// the host spatial_sort's key (abi.cpp), from the current positions
__global__ void k_morton_keys(int64_t n, const double4* __restrict__ pos, Box b, int nx, int ny,
                              int nz, uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double4 p = pos[s];
  const int cx = min(nx - 1, (int)(p.x / b.lx * nx));
  const int cy = min(ny - 1, (int)(p.y / b.ly * ny));
  const int cz = min(nz - 1, (int)(p.z / b.lz * nz));
  key[s] = spread3_dev(cx) | spread3_dev(cy) << 1 | spread3_dev(cz) << 2;
  val[s] = (int32_t)s;
}

// Molecule-keyed order (sites of a molecule consecutive, molecules in
// Morton order, so a 3-site cluster of cluster.cu is one water): the key of
// a site is the Morton key of its molecule's representative site `rep`, then
// rep itself (ties of two molecules in one cell stay apart). rep: the given
// array (the first molecule sort, abi.cpp), or else the first site of the
// site's run of equal molecule ids in the current order (the order already
// molecule-keyed: runs are molecules). The key needs the cell code in 33
// bits (<= 2048 cells per edge; checked by the caller).
__global__ void k_morton_keys_mol(int64_t n, const double4* __restrict__ pos,
                                  const int32_t* __restrict__ mol,
                                  const int32_t* __restrict__ rep_in, Box b, int nx, int ny,
                                  int nz, uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  int64_t r = s;
  if (rep_in) {
    r = rep_in[s];
  } else {
    const int32_t m = mol[s];
    for (int k = 0; k < 64 && r > 0 && mol[r - 1] == m; ++k) --r;
  }
  const double4 p = pos[r];
  const int cx = min(nx - 1, (int)(p.x / b.lx * nx));
  const int cy = min(ny - 1, (int)(p.y / b.ly * ny));
  const int cz = min(nz - 1, (int)(p.z / b.lz * nz));
  key[s] = (spread3_dev(cx) | spread3_dev(cy) << 1 | spread3_dev(cz) << 2) << 31 | (uint64_t)r;
  val[s] = (int32_t)s;
}

__global__ void k_inverse(int64_t n, const int32_t* __restrict__ ord, int32_t* __restrict__ inv) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) inv[ord[s]] = (int32_t)s;
}

// dst[s * K + k] = src[ord[s] * K + k]
template <class T, int K>
__global__ void k_permute(int64_t n, const int32_t* __restrict__ ord, const T* __restrict__ src,
                          T* __restrict__ dst) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t o = ord[s];
#pragma unroll
  for (int k = 0; k < K; ++k) dst[s * K + k] = src[o * K + k];
}

// index arrays: v <- inv[v] (entries in [0, n)); codes: (inv[v >> 1] << 1) | (v & 1)
__global__ void k_remap(int64_t m, const int32_t* __restrict__ inv, int32_t* __restrict__ v,
                        int code) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int32_t x = v[k];
  v[k] = code ? ((inv[x >> 1] << 1) | (x & 1)) : inv[x];
}

// frames: (type, zatom, xatom, 0) with the atoms remapped
__global__ void k_remap_frames(int64_t n, const int32_t* __restrict__ inv, int4* __restrict__ f) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  int4 v = f[s];
  if (v.x != 0) {
    v.y = inv[v.y];
    v.z = inv[v.z];
  }
  f[s] = v;
}

// CSR rows permuted with the sites: counts of the new order
__global__ void k_csr_counts(int64_t n, const int32_t* __restrict__ ord,
                             const int32_t* __restrict__ start, int32_t* __restrict__ cnt) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < n) cnt[s] = start[ord[s] + 1] - start[ord[s]];
  if (s == n) cnt[s] = 0;
}

__global__ void k_csr_copy(int64_t n, const int32_t* __restrict__ ord,
                           const int32_t* __restrict__ ostart, const int32_t* __restrict__ olist,
                           const int32_t* __restrict__ nstart, int32_t* __restrict__ nlist,
                           const int32_t* __restrict__ inv, int code) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int32_t o = ord[s];
  const int32_t a = ostart[o], m = ostart[o + 1] - a, b = nstart[s];
  for (int32_t k = 0; k < m; ++k) {
    const int32_t x = olist[a + k];
    nlist[b + k] = code ? ((inv[x >> 1] << 1) | (x & 1)) : inv[x];
  }
}

namespace {

struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t b) {
    if (b > bytes) {
      cudaFree(p);
      p = nullptr;
      MDG_CUDA_CHECK(cudaMalloc(&p, b));
      bytes = b;
    }
    return p;
  }
  ~Scratch() { cudaFree(p); }
};

template <class T, int K>
void permute_array(mdg_ctx* c, const int32_t* ord, T* arr, void* tmp) {
  if (!arr) return;
  const int64_t n = c->n;
  MDG_LAUNCH(c, "resort_permute", grid_for(n, 256), 256, 0, (k_permute<T, K>), n, ord, arr,
             (T*)tmp);
  MDG_CUDA_CHECK(cudaMemcpyAsync(arr, tmp, (size_t)n * K * sizeof(T), cudaMemcpyDeviceToDevice,
                                 c->stream));
}

// a CSR (start[n + 1], list) rebuilt in the new order, entries remapped
void permute_csr(mdg_ctx* c, const int32_t* ord, const int32_t* inv, int32_t* start,
                 int32_t* list, int code, Scratch& s1, Scratch& s2, Scratch& s3) {
  if (!start || !list) return;
  const int64_t n = c->n;
  int32_t total = 0;
  MDG_CUDA_CHECK(cudaMemcpyAsync(&total, start + n, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  int32_t* cnt = (int32_t*)s1.get((n + 1) * sizeof(int32_t));
  int32_t* nstart = (int32_t*)s2.get((n + 1) * sizeof(int32_t));
  int32_t* nlist = (int32_t*)s3.get(std::max<int32_t>(total, 1) * sizeof(int32_t));
  MDG_LAUNCH(c, "resort_csr_counts", grid_for(n + 1, 256), 256, 0, k_csr_counts, n, ord, start,
             cnt);
  size_t tb = 0;
  MDG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, nstart, n + 1, c->stream));
  static thread_local Scratch st;
  MDG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(st.get(tb), tb, cnt, nstart, n + 1, c->stream));
  MDG_LAUNCH(c, "resort_csr_copy", grid_for(n, 256), 256, 0, k_csr_copy, n, ord, start, list,
             nstart, nlist, inv, code);
  MDG_CUDA_CHECK(cudaMemcpyAsync(start, nstart, (n + 1) * sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, c->stream));
  if (total > 0)
    MDG_CUDA_CHECK(cudaMemcpyAsync(list, nlist, total * sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, c->stream));
}

}  // namespace

bool mol_order_fits(const mdg_ctx* c) {
  const int nx = std::max(1, (int)(c->lx / 2.0)), ny = std::max(1, (int)(c->ly / 2.0)),
            nz = std::max(1, (int)(c->lz / 2.0));
  return c->n < ((int64_t)1 << 31) && std::max(nx, std::max(ny, nz)) <= 2048;
}

void resort_sites(mdg_ctx* c, const int32_t* rep) {
  // a domain's owned and halo parts are each re-ordered in place (owned
  // sites first); only before its group exists (the halo maps are in sorted
  // indices)
  if (c->group || (c->n_own != c->n && !rep))
    throw_error(MDG_CONTRACT, "resort: not for a domain in a group (halo maps use sorted indices)");
  const int64_t n = c->n;
  if (n < 2) return;
  const bool molkey = (rep || c->mol_sorted) && mol_order_fits(c);
  static thread_local Scratch sk, sv, sk2, sv2, sinv, stmp, scub, c1, c2, c3;
  uint64_t* key = (uint64_t*)sk.get(n * sizeof(uint64_t));
  int32_t* val = (int32_t*)sv.get(n * sizeof(int32_t));
  uint64_t* key2 = (uint64_t*)sk2.get(n * sizeof(uint64_t));
  int32_t* ord = (int32_t*)sv2.get(n * sizeof(int32_t));
  int32_t* inv = (int32_t*)sinv.get(n * sizeof(int32_t));
  const int nx = std::max(1, (int)(c->lx / 2.0)), ny = std::max(1, (int)(c->ly / 2.0)),
            nz = std::max(1, (int)(c->lz / 2.0));
  if (molkey)
    MDG_LAUNCH(c, "resort_keys", grid_for(n, 256), 256, 0, k_morton_keys_mol, n, c->pos, c->mol,
               rep, make_box(c->lx, c->ly, c->lz), nx, ny, nz, key, val);
  else
    MDG_LAUNCH(c, "resort_keys", grid_for(n, 256), 256, 0, k_morton_keys, n, c->pos,
               make_box(c->lx, c->ly, c->lz), nx, ny, nz, key, val);
  // owned sites, then the halo, each sorted by its keys
  const int64_t parts[2][2] = {{0, c->n_own}, {c->n_own, n}};
  for (const auto& pr : parts) {
    const int64_t m = pr[1] - pr[0];
    if (m <= 0) continue;
    size_t tb = 0;
    MDG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key + pr[0], key2 + pr[0],
                                                   val + pr[0], ord + pr[0], (int)m, 0, 64,
                                                   c->stream));
    MDG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(scub.get(tb), tb, key + pr[0], key2 + pr[0],
                                                   val + pr[0], ord + pr[0], (int)m, 0, 64,
                                                   c->stream));
  }
  MDG_LAUNCH(c, "resort_inverse", grid_for(n, 256), 256, 0, k_inverse, n, ord, inv);
  void* tmp = stmp.get((size_t)n * 3 * sizeof(double4));
  // per-site records
  permute_array<double4, 1>(c, ord, c->pos, tmp);
  permute_array<double4, 1>(c, ord, c->vsite, tmp);
  permute_array<double4, 1>(c, ord, c->vdwp, tmp);
  permute_array<double4, 1>(c, ord, c->pq4, tmp);
  permute_array<double2, 1>(c, ord, c->polp, tmp);
  permute_array<int32_t, 1>(c, ord, c->vtype, tmp);
  permute_array<int32_t, 1>(c, ord, c->mol, tmp);
  permute_array<double, 1>(c, ord, c->hfac, tmp);
  permute_array<double4, 3>(c, ord, c->mp, tmp);
  permute_array<int32_t, 1>(c, ord, c->d_perm, tmp);
  if (c->has_vel) permute_array<double4, 1>(c, ord, c->vel, tmp);
  // results of the last step stay fetchable
  for (double4* v : {c->force, c->torque, c->mu, c->eperm})
    permute_array<double4, 1>(c, ord, v, tmp);
  // the ASPC history of converged dipoles (mdg_md_run)
  for (int j = 0; j < c->aspc_count; ++j)
    permute_array<double4, 1>(c, ord, c->aspc_hist + (size_t)j * c->n_cap, tmp);
  if (c->has_frames) {
    permute_array<double4, 3>(c, ord, c->mploc, tmp);
    permute_array<int4, 1>(c, ord, c->frame, tmp);
    MDG_LAUNCH(c, "resort_frames", grid_for(n, 256), 256, 0, k_remap_frames, n, inv, c->frame);
    permute_csr(c, ord, inv, c->fref_start, c->fref, 1, c1, c2, c3);
  }
  // site indices held in arrays
  permute_array<int32_t, 1>(c, ord, c->hpar, tmp);
  MDG_LAUNCH(c, "resort_remap", grid_for(n, 256), 256, 0, k_remap, n, inv, c->hpar, 0);
  MDG_LAUNCH(c, "resort_remap", grid_for(n, 256), 256, 0, k_remap, n, inv, c->d_iperm, 0);
  permute_csr(c, ord, inv, c->child_start, c->child, 0, c1, c2, c3);
  permute_csr(c, ord, inv, c->excl_start, c->excl, 0, c1, c2, c3);
  if (c->nbonds > 0)
    MDG_LAUNCH(c, "resort_remap", grid_for(2 * c->nbonds, 256), 256, 0, k_remap, 2 * c->nbonds,
               inv, (int32_t*)c->bond_ij, 0);
  if (c->nangles > 0)  // (i, j, k, 0): the pad word is 0, a valid index
    MDG_LAUNCH(c, "resort_remap", grid_for(4 * c->nangles, 256), 256, 0, k_remap,
               4 * c->nangles, inv, (int32_t*)c->angle_ijk, 0);
  // host copies of the maps
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->perm.data(), c->d_perm, n * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, c->stream));
  MDG_CUDA_CHECK(cudaMemcpyAsync(c->iperm.data(), c->d_iperm, n * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, c->stream));
  MDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  // everything in sorted indices is stale: lists, buffered rows, pruned rows
  for (auto& L : c->lists) {
    L.valid = false;
    L.inner.src_version = -1;
    L.inner.ubuilt = false;
  }
  c->plist.valid = false;
  c->plist.cl_valid = false;
  c->plist.ubuilt = false;
  c->fout_seq = 0;
  c->mol_sorted = molkey;
}

}  // namespace mdg
