// debug.cu -- list invariants checked on the device in debug builds
// (make -C paper_1906_01211_b200 debug -> libmdg_debug.so, -DMDG_DEBUG).
// Every row a kernel walks: count within [0, cap], every neighbour index in
// [0, n_all) and not the row's own site, strictly ascending (flag bit masked)
// when the row set claims to be sorted. A violation is a device assert
// (cudaErrorAssert from the next call), so the parity suite run against the
// debug library doubles as a bounds check of the product's indexing.
#include "common.cuh"

namespace mdg {

#ifdef MDG_DEBUG
__global__ void k_dbg_rows(int64_t rows, int64_t n_all, const int32_t* __restrict__ nbr,
                           const int32_t* __restrict__ cnt, int32_t cap, int sorted) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int c = cnt[i];
  assert(c >= 0 && c <= cap);
  const int32_t* row = nbr + (size_t)i * cap;
  int32_t prev = -1;
  for (int k = 0; k < c; ++k) {
    const int32_t j = row[k] & 0x7fffffff;
    assert(j >= 0 && j < n_all);
    assert(j != (int32_t)i);
    if (sorted) assert(j > prev);
    prev = j;
  }
}
#endif

void debug_check_rows(mdg_ctx* c, const char* what, const int32_t* nbr, const int32_t* cnt,
                      int32_t cap, int64_t rows, int64_t n_all, bool sorted) {
#ifdef MDG_DEBUG
  if (rows <= 0) return;
  MDG_LAUNCH(c, "dbg_rows", grid_for(rows, 128), 128, 0, k_dbg_rows, rows, n_all, nbr, cnt,
             cap, sorted ? 1 : 0);
  cuda_check(cudaStreamSynchronize(c->stream), what);
#else
  (void)c, (void)what, (void)nbr, (void)cnt, (void)cap, (void)rows, (void)n_all, (void)sorted;
#endif
}

}  // namespace mdg
