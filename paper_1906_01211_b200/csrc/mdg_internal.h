// mdg_internal.h -- context, device layout and shared device helpers.
//
// Device data layout (HBM, all in the context's spatially sorted order):
//   pos    double4[n]   x, y, z, exclusion group (as double; one sector,
//                       so the pair prologues need no second gather)
//   vsite  double4[n]   Halgren-reduced x, y, z, exclusion group (vdW lists)
//   vdwp   double4[n]   lj_sigma, sqrt(lj_eps), hal_r0, sqrt(hal_eps)
//   polp   double2[n]   polarizability, polarizability^(1/6)
//   mol    int32[n]     exclusion group
//   mp     double4[3n]  (mux,muy,muz,Qxx) (Qxy,Qxz,Qyy,Qyz) (Qzz,0,0,0)
//   lists  row-major:   nbr[i*cap + k] = j (cap a multiple of 32), cnt[i]
//                       neighbours (both directions) within the list cutoff
//   vectors (forces, fields, dipoles, CG) double4[n], w unused.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "../../include/mdg.h"

namespace mdg {

#ifndef MDG_BLOCK
#define MDG_BLOCK 128
#endif
constexpr int kBlock = MDG_BLOCK;
constexpr int kAspcDepth = 6;  // ASPC k = 4
constexpr int kCl = 3;         // sites per cluster (cluster.cu): one water molecule
constexpr int kStaleSlot = 120;  // results 120..123: list l outdated (nlist.cu)  // pair-kernel block: 4 warps = 4 site groups
constexpr int kRedVals = 16;     // per-block partial slots (energies + virial)
// device result slots: 0-9 nonpolar, 10-19 multipoles, 20-27 PCG, 30 Jacobi,
// 40 polarization energy, 50-51 count_within, 60-65 list stats,
// 70-79 polarization forces (pair energy, virial), 80-97 PME (pme.cu)
constexpr int kResultSlots = 128;
constexpr int kMaxBlocksRed = 1 << 20;

struct Box {
  double lx, ly, lz, ix, iy, iz, hx, hy, hz;
};

inline Box make_box(double lx, double ly, double lz) {
  // host-computed reciprocals and halves, as proj/src/kernels_scalar.cpp:16-17
  return Box{lx, ly, lz, 1.0 / lx, 1.0 / ly, 1.0 / lz, 0.5 * lx, 0.5 * ly, 0.5 * lz};
}

struct Grid {
  int ncx, ncy, ncz;
  double ex, ey, ez;
};

struct DevList {
  bool valid = false;
  double cutoff = 0;
  int sites = 0;
  int32_t cap = 0;              // ELL width (slots per site)
  int32_t* nbr = nullptr;
  int32_t* cnt = nullptr;
  double4* ref0 = nullptr;      // site positions at the build (staleness check)
  size_t nbr_elems = 0;
  int64_t half_pairs = 0;
  int32_t max_cnt = 0;
  int64_t version = 0;          // bumped by every (re)build / import
  bool sorted = false;          // every row ascending in j
  // Buffered inner list (dynamic pruning): the rows cut to kernel cutoff + a
  // buffer b, valid while no site has moved more than b/2 since the cut
  // (checked on the device every call; the cut is redone when it fails).
  struct Inner {
    double rc = 0;                // cut radius (kernel cutoff + buffer)
    int64_t src_version = -1;     // source list version it was cut from
    int32_t* nbr = nullptr;
    int32_t* cnt = nullptr;
    size_t elems = 0;
    double4* ref = nullptr;       // site positions at the cut
    int32_t* flag = nullptr;      // device: 1 = cut again (motion), 2 = forced (new list)
    int32_t* gen = nullptr;       // device: cuts done (the cluster unions' staleness test)
    // cuts done, counted by the cut kernel in mapped page-locked memory (read
    // by the host without a sync): when most calls need a new cut (sites
    // moving fast), the buffer only adds a pass, so the rows are bypassed
    int32_t* hcuts = nullptr;
    int32_t* dcuts = nullptr;
    int calls = 0, cuts0 = 0, bypass = 0;
    bool cut_sorted = true;  // the last cut sorted its rows (kernel_rows want_sorted)
    // site-cluster unions of these rows (cluster.cu build_row_unions): per
    // cluster of kCl consecutive sites the sorted union of their rows,
    // rebuilt on the device when the rows are cut again
    int32_t* uidx = nullptr;
    int32_t* ucnt = nullptr;
    int32_t* ugen = nullptr;
    size_t uelems = 0;
    int64_t ucnt_elems = 0;
    int32_t ucap = 0;
    int64_t ncl = 0;
    uintptr_t ukey[3] = {0, 0, 0};
    bool ubuilt = false;
  } inner;
};

// Pruned list: the pairs of a source list within a kernel cutoff, compacted
// per site (same sliced-ELL layout), j | 0x80000000 when i, j share a
// molecule; trr holds the Ewald/Thole T pair tensor (rr3, rr5) per slot.
// one 32-entry chunk of a cluster's stream (cluster.cu): the entries' pair
// tensors per cluster site, then their indices -- one bulk copy of 1664 B
struct ClChunk {
  double2 ten[kCl][32];
  int32_t idx[32];
};

struct PrunedList {
  bool valid = false;
  int src = -1;
  double cutoff = 0;
  int32_t cap = 0;
  int32_t* nbr = nullptr;
  int32_t* cnt = nullptr;
  double2* trr = nullptr;
  size_t elems = 0;
  int64_t directed = 0;
  bool sorted = false;  // rows ascending in (j & 0x7fffffff) (source sorted)
  // site clusters (cluster.cu): kCl consecutive sites (a water molecule in
  // the molecule-keyed order). Per cluster, nch chunks (ClChunk) hold U75,
  // the sorted union of the sites' buffered inner rows (indices), and per
  // site the pair tensors (rr3, rr5) with each entry -- written by the field
  // pass every step through cmap[i * mstride + h] (the U75 position of slot
  // h of site i's row), zero beyond the cutoff or when the entry is not in
  // the site's row. The unions and maps are rebuilt when the rows are cut.
  bool cl_valid = false;
  int64_t ncl = 0;
  int32_t* ucnt = nullptr;
  int32_t* ugen = nullptr;  // device: inner-row generation the unions were built from
  int64_t ucnt_elems = 0;
  double ucut = 0.0;
  uintptr_t ukey[4] = {0, 0, 0, 0};
  uint16_t* cmap = nullptr;
  size_t melems = 0;
  int32_t mstride = 0;  // rows.cap of the mapped rows
  int32_t tcap = 0;     // entries per cluster (nch * 32)
  int32_t nch = 0;
  ClChunk* cst = nullptr;
  size_t celems = 0;    // chunks allocated
  bool ubuilt = false;  // the union buffers hold the unions of the keyed rows
};

// arguments of the cluster mat-vec (cluster.cu)
struct CLArgs {
  int64_t n;    // owned sites
  int64_t ncl;  // clusters
  int ipw;      // clusters per block (MDG_LAUNCH_SITES)
  const double4* __restrict__ pos;
  const double2* __restrict__ polp;
  const ClChunk* __restrict__ cst;   // [ncl][nch]
  const int32_t* __restrict__ ucnt;  // [ncl] entries
  int32_t nch;
  Box b;
  const double4* __restrict__ in;
  double4* __restrict__ out;
  double* __restrict__ partials;
  const double* __restrict__ res;  // PCG: result slots (converged flag 27)
};

// Communication of a multi-domain PCG solve (group.cu): refresh the halo of
// a device vector in every local domain, and sum result slots over all
// domains, both ordered on the domains' stream.
struct PcgComm {
  virtual ~PcgComm() = default;
  virtual void exchange(int vec_id) = 0;
  virtual void allreduce(int slot, int nv) = 0;
  virtual bool capturable() const = 0;  // all ops may sit in a while graph
  virtual int64_t n_global() const = 0;
  virtual uintptr_t generation() const = 0;  // changes with the halo plans
  // Interior/halo overlap: exchange_begin issues the refresh on the group's
  // communication stream (after everything queued so far on the domains'
  // stream), exchange_end makes the domains' stream wait for it; between the
  // two, the mat-vec of the sites whose rows hold no halo site runs.
  // replicated-grid reciprocal space (pme.cu PmeDoms): sum the domains'
  // grids (count doubles each). grid_shared: one device, the sum lands in
  // grids[0] and every domain reads it; else each rank's grid is all-reduced
  // in place. recip_root: the domain that carries the convolution energy.
  virtual void grid_sum(double* const* grids, int n, size_t count) {}
  virtual bool grid_shared() const { return false; }
  virtual bool recip_root(int dom) const { return dom == 0; }
  virtual bool overlap() const { return false; }
  // slab-decomposed reciprocal space (pme.cu PmeDoms, MDG_PME_SLAB=1):
  // slab_parts() parts (0: the replicated grid above), local domain d is
  // part slab_part(d). grids / bufs: the LOCAL domains' buffers, in domain
  // order. slab_reduce: part p's grid holds, in its planes [off[p],
  // off[p+1]) (doubles), the sum of every domain's grid. slab_alltoall: part
  // p's src[soff[p*P+q], +cnt[p*P+q]) lands in part q's dst at
  // doff[q*P+p] (complex counts). slab_allgather: every local grid (one per
  // device) holds every part's planes.
  virtual int slab_parts() const { return 0; }
  virtual int slab_part(int dom) const { return dom; }
  virtual void slab_reduce(double* const* grids, int n, const int64_t* off) {}
  virtual void slab_alltoall(cufftDoubleComplex* const* src, cufftDoubleComplex* const* dst,
                             int n, const int64_t* soff, const int64_t* doff,
                             const int64_t* cnt) {}
  virtual void slab_allgather(double* const* grids, int n, const int64_t* off) {}
  virtual void exchange_begin(int vec_id) { exchange(vec_id); }
  virtual void exchange_end() {}
};

// reciprocal-space Ewald in the AMOEBA step (mdg_set_ewald_recip): grid,
// B-spline order, the step's alpha (set per call), excluded pairs removed
struct PolarRecip {
  int k1 = 0, k2 = 0, k3 = 0, order = 0;
  double alpha = 0.0, electric = 1.0;
  bool exclude = true;
  bool on() const { return k1 > 0; }
};

struct ProfEntry {
  int64_t count = 0;
  double ms = 0;
};

struct PendingEvent {
  std::string name;
  cudaEvent_t a, b;
};

}  // namespace mdg

constexpr int kMaxVdwTypes = 64;
struct mdg_group;

struct mdg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n_cap = 0;
  int32_t max_pairs = 0;

  // system: sites [0, n_own) are owned (their rows are computed), sites
  // [n_own, n) are the halo of a spatial domain (inputs only); single-domain
  // runs have n_own == n. n_global counts all sites of all domains.
  int64_t n = 0;
  int64_t n_own = 0;
  int64_t n_global = 0;
  // the domain group this context belongs to (group.cu; NULL: single domain)
  mdg_group* group = nullptr;
  // interior / boundary split of the owned sites (domain groups with
  // interior/halo overlap): boundary sites (a halo site in their pruned row)
  // first, then the interior ones; dd_nsel = number of boundary sites
  int32_t* dd_sites = nullptr;
  uint8_t* dd_flags = nullptr;
  int* dd_nsel = nullptr;
  void* dd_tmp = nullptr;
  size_t dd_tmp_bytes = 0;
  int32_t* d_iperm = nullptr;  // caller -> sorted index
  int32_t* d_idx = nullptr;    // staging for halo index lists
  double lx = 0, ly = 0, lz = 0;
  bool has_system = false, has_mpoles = false, has_hred = false, has_mol = false;
  std::vector<int32_t> perm;   // sorted -> caller index
  std::vector<int32_t> iperm;  // caller -> sorted index

  // device arrays (sorted order)
  int32_t* d_perm = nullptr;
  double4* pos = nullptr;
  double4* vsite = nullptr;
  double4* vdwp = nullptr;
  // Site parameter types: when the system has <= kMaxVdwTypes distinct
  // (sigma, eps_lj, r0, eps_hal, charge, polarizability) tuples, vtab[t] /
  // ptab[t] hold the vdwp / pq4 records of a representative site and the type rides in the high word of
  // pos.w / vsite.w, so the LJ / Halgren bodies read j's parameters from a
  // table every lane shares instead of a 32-B gather per pair (charges and
  // Thole factors likewise from ptab).
  int32_t* vtype = nullptr;
  double4* vtab = nullptr;
  double4* ptab = nullptr;  // pq4 record of each type's representative site
  int n_vtypes = 0;  // 0: per-site parameters (vdwp gathers)
  double2* polp = nullptr;
  double4* pq4 = nullptr;  // (polarizability, polarizability^(1/6), charge, alpha^(-1/6))
  int32_t* mol = nullptr;
  int32_t* hpar = nullptr;
  double* hfac = nullptr;
  int32_t* child_start = nullptr;  // CSR of Halgren children per parent
  int32_t* child = nullptr;
  double4* mp = nullptr;
  // local multipole frames (frames.cu): (type, zatom, xatom, 0) per site,
  // local-frame multipoles (mp layout), per-site frame forces (i, z, x) and
  // the CSR of frame references per atom (2 * site + role)
  bool has_frames = false;
  // same-molecule partners per site (CSR, sorted indices): PME's removal of
  // the excluded pairs from the reciprocal sum
  int32_t* excl_start = nullptr;
  int32_t* excl = nullptr;
  void* pme = nullptr;      // PmeState (pme.cu): charges / permanent multipoles
  void* pme_pol = nullptr;  // PmeState of the polarization fields (main stream)
  mdg::PolarRecip pol_recip;  // mdg_set_ewald_recip
  bool recip_in_step = false;  // last AMOEBA step added the multipole PME terms
  // MD (md.cu): velocities (w = 1/mass) and harmonic bonded terms
  double4* vel = nullptr;
  double4* fbond = nullptr;  // inner-level (bonded) forces of BAOAB-RESPA
  int64_t md_rebuilds = 0;   // list rebuilds inside mdg_md_run (re-sort cadence)
  // early warning of list staleness (nlist.cu): set by the device when a site
  // has moved more than 0.6 x the tolerable motion since its list was built;
  // mapped page-locked memory, read by mdg_md_run without a sync to rebuild
  // ahead of schedule
  int32_t* h_warn = nullptr;
  int32_t* d_warn = nullptr;
  int32_t list_gen = 0;  // bumped by every list build: the warning names the lists it is about
  // ASPC dipole predictor of mdg_md_run (polar.cu k_mu0_aspc): a ring of the
  // last kAspcDepth converged dipole vectors (n_cap each)
  bool aspc_on = false;
  double4* aspc_hist = nullptr;
  int aspc_head = 0, aspc_count = 0;
  bool has_vel = false;
  int2* bond_ij = nullptr;
  double2* bond_par = nullptr;  // (k, r0)
  int4* angle_ijk = nullptr;    // (i, vertex j, k, 0)
  double2* angle_par = nullptr; // (k, theta0)
  int64_t nbonds = 0, nangles = 0;
  int4* frame = nullptr;
  double4* mploc = nullptr;
  double4* fbuf = nullptr;
  int32_t* fref_start = nullptr;
  int32_t* fref = nullptr;

  // cell grid scratch
  int32_t* cell_of = nullptr;
  int32_t* cell_start = nullptr;
  int32_t* cell_fill = nullptr;
  int32_t* cell_atoms = nullptr;
  int64_t cell_cap = 0;
  int32_t* d_flag = nullptr;  // device error/overflow flags [8]

  // vectors
  double4* force = nullptr;
  double4* force2 = nullptr;
  double4* torque = nullptr;
  double4* field = nullptr;
  double4* eperm = nullptr;
  double4* mu = nullptr;
  double4* cg_r = nullptr;
  double4* cg_z = nullptr;
  double4* cg_p = nullptr;
  double4* cg_q = nullptr;
  double4* vin = nullptr;  // generic input vector (dipoles for tmatvec)

  // reductions
  double* partials = nullptr;
  int64_t partial_blocks = 0;
  double* results = nullptr;    // device result slots
  double* h_results = nullptr;  // pinned mirror

  // staging
  double* h_stage = nullptr;
  double* d_stage = nullptr;
  size_t stage_bytes = 0;

  mdg::DevList lists[MDG_MAX_LISTS];
  mdg::PrunedList plist;
  int64_t epoch = 0;  // source of DevList::version
  // full-row (bitwise reproducible) pair sums instead of half rows + atomics
  bool deterministic = false;
  // fault injection (mdg_set_debug_perturb): added to the first returned
  // force component and energy, so the parity checks' failure path is tested
  double debug_perturb = 0.0;
  bool overlap = true;  // AMOEBA step on two streams (mdg_set_overlap)
  // PCG on site clusters (cluster.cu; mdg_set_cluster_matvec, MDG_CLUSTER_MATVEC)
  bool cluster_matvec = false;
  // Halgren on site clusters (nonpolar.cu k_halgren_cl; MDG_CLUSTER_HALGREN)
  bool cluster_halgren = true;
  // site order molecule-keyed (resort.cu): a molecule's sites consecutive
  bool mol_sorted = false;
  bool has_polar_force = false;  // last AMOEBA step added polarization forces
  // second stream of the AMOEBA step: Halgren + multipoles run beside the
  // permanent field + PCG (independent work); its own block partials
  cudaStream_t aux_stream = nullptr;
  double* aux_partials = nullptr;
  int64_t aux_partial_blocks = 0;
  cudaEvent_t ev_fork = nullptr, ev_tpre = nullptr, ev_join = nullptr;
  // registered page-locked force outputs (mdg_set_force_output): the step
  // DMAs caller-order forces into them as soon as they are final
  double* fout[3] = {nullptr, nullptr, nullptr};
  double* d_fout = nullptr;    // 3 n doubles, caller order
  uint64_t fout_seq = 0;       // API call sequence number of the step that queued it

  // last step
  double energies[4] = {0, 0, 0, 0};
  double virial[9] = {0};
  int64_t pcg_iters = 0;
  double pcg_rms = 0;

  // instrumentation
  int64_t launches = 0;
  bool profile = false;
  std::map<std::string, mdg::ProfEntry> prof;
  std::vector<mdg::PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t timer_a = nullptr, timer_b = nullptr;
  int64_t last_grid = 0;  // blocks of the last MDG_LAUNCH_SITES launch
  // shape overrides for MDG_LAUNCH_SITES (0: occupancy limit, 16 waves):
  // resident blocks per SM and waves, so two streams can share every SM
  int launch_bps = 0, launch_waves = 0;
};

namespace mdg {

// ---- error handling -----------------------------------------------------
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void throw_error(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define MDG_CUDA_CHECK(x) ::mdg::cuda_check((x), #x)

// ---- launch bookkeeping -------------------------------------------------
void launch_begin(mdg_ctx* c, const char* name);
void launch_end(mdg_ctx* c, const char* name);
void flush_profile(mdg_ctx* c);

#define MDG_LAUNCH(ctx, name, grid, block, smem, kernel, ...)                  \
  do {                                                                         \
    ::mdg::launch_begin((ctx), (name));                                        \
    kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);           \
    ::mdg::launch_end((ctx), (name));                                          \
  } while (0)

inline unsigned grid_for(int64_t n, int block = kBlock) {
  return (unsigned)((n + block - 1) / block);
}

// Warp-per-site kernels run exactly one wave: (#SMs x resident blocks per
// SM) blocks, each walking a contiguous (Morton-ordered, spatially compact)
// range of sites with its warps interleaved, so an SM's live neighbour data
// is a sliding window that stays in L1. Returns sites per block.
int64_t sites_per_block(const void* kernel, int64_t n, int bps_cap = 0, int waves = 0);

// Launch a warp-per-site kernel whose args struct has `ipw` (sites per block)
// and `partials`; records the grid in ctx->last_grid for the finalize.
#define MDG_LAUNCH_SITES(ctx, name, n, args, kernel)                             \
  do {                                                                         \
    const int64_t _ipb = ::mdg::sites_per_block((const void*)(kernel), (n), (ctx)->launch_bps, (ctx)->launch_waves);   \
    (args).ipw = (int)_ipb;                                                    \
    const int64_t _g = ((n) + _ipb - 1) / _ipb;                                \
    ::mdg::ensure_partials((ctx), _g);                                         \
    (args).partials = (ctx)->partials;                                         \
    (ctx)->last_grid = _g;                                                     \
    MDG_LAUNCH((ctx), (name), (unsigned)_g, ::mdg::kBlock, 0, kernel, (args)); \
  } while (0)

inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// Launches inside this scope go to the context's aux stream with its own
// partials buffer (no-op when !on).
struct AuxScope {
  mdg_ctx* c;
  bool on;
  cudaStream_t s;
  double* p;
  int64_t pb;
  int bps = 0, waves = 0;
  AuxScope(mdg_ctx* c_, bool on_) : c(c_), on(on_) {
    if (!on) return;
    static const int aux_bps = env_int("MDG_AUX_BPS", 0);
    static const int aux_waves = env_int("MDG_AUX_WAVES", 0);
    bps = c->launch_bps;
    waves = c->launch_waves;
    c->launch_bps = aux_bps;
    c->launch_waves = aux_waves;
    s = c->stream;
    p = c->partials;
    pb = c->partial_blocks;
    c->stream = c->aux_stream;
    c->partials = c->aux_partials;
    c->partial_blocks = c->aux_partial_blocks;
  }
  ~AuxScope() {
    if (!on) return;
    c->aux_partials = c->partials;
    c->aux_partial_blocks = c->partial_blocks;
    c->stream = s;
    c->partials = p;
    c->partial_blocks = pb;
    c->launch_bps = bps;
    c->launch_waves = waves;
  }
  AuxScope(const AuxScope&) = delete;
  AuxScope& operator=(const AuxScope&) = delete;
};

// ---- host entry points implemented in the .cu files -----------------------
void ensure_partials(mdg_ctx* c, int64_t blocks);
// Sum per-block partials [blocks][kRedVals] in fixed order into
// results[slot .. slot+nvals), scaled by `scale`.
void finalize_partials(mdg_ctx* c, int64_t blocks, int nvals, int slot, double scale);
void fetch_results(mdg_ctx* c);

void nlist_build(mdg_ctx* c, int list_id, double list_cutoff, int sites);
// max and sum of per-site counts -> results[slot], results[slot + 1]
void count_stats(mdg_ctx* c, const int32_t* cnt, int slot);

struct NonpolarArgs {
  int do_lj, do_coul, shift, exclude;
  double cutoff, alpha, electric;
};
// Writes c->force (sorted), energies into results[0] (lj) and results[1]
// (coulomb), virial into results[2..10].
void run_nonpolar(mdg_ctx* c, int list_id, const NonpolarArgs& a);
// Halgren on list (atomic or reduced sites); writes c->force (atoms),
// results[0] energy, results[2..10] virial.
void run_halgren(mdg_ctx* c, int list_id, double cutoff, double delta, double gamma,
                 int exclude);
// E = T v (c->vin -> out), alpha >= 0.
void run_tmatvec(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                 const double4* in, double4* out);
void run_perm_field(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                    int exclude, double4* out);
// Returns iterations; throws CONVERGENCE (with last_rms set) on failure.
int64_t run_pcg(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                double tol_debye, int64_t max_iter, double* last_rms);
int64_t run_jacobi(mdg_ctx* c, int list_id, double cutoff, double thole_a, double tol,
                   int64_t max_iter, double* last_resid);
void run_mpole(mdg_ctx* c, int list_id, double alpha, double cutoff, double electric,
               int exclude, bool accumulate);
// multipoles over the pruned list (c->plist)
void run_mpole_pruned(mdg_ctx* c, double alpha, double electric, int exclude, bool accumulate);
// One pass over list_id: prune to `cutoff` into c->plist (exclusion flag in
// bit 31), store the Ewald/Thole T pair tensors in c->plist.trr, and write
// the permanent field into c->eperm.
void run_field_tpre(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                    int exclude);
// Cluster unions (U75) of the rows the field pass walks, their slot maps
// and the zero tensors of the slots no row fills (cluster.cu); rebuilt on the
// device when `gen` (the rows' cut generation) moved, unconditionally when
// `force`. tcap: the entry capacity per cluster, a multiple of 32 (entries
// past it are counted, not stored: the caller retries larger). Returns false when the
// cluster path does not apply.
bool build_clusters(mdg_ctx* c, double cutoff, const struct ListView& rows, const int32_t* gen,
                    int32_t tcap, bool force);
void count_stats_n(mdg_ctx* c, const int32_t* cnt, int64_t n, int slot);
// The cluster unions of list `list_id`'s buffered rows `rows` (L.inner), for
// the cluster pair kernels (Halgren); false when they do not apply (rows not
// buffered, deterministic mode, disabled)
bool build_row_unions(mdg_ctx* c, int list_id, const struct ListView& rows);
// an NCCL / LOCAL group runs the interior/halo overlapped exchange (per-site rows)
bool group_overlap(const mdg_ctx* c);
CLArgs cl_args(mdg_ctx* c, const double4* in, double4* out);
const void* cl_matvec_kernel(bool pcg);
void cl_matvec_launch(mdg_ctx* c, CLArgs& k, bool pcg, const char* name);
void cl_matvec_launch_raw(const CLArgs& k, unsigned grid, cudaStream_t s);
// PCG on the precomputed T tensors of c->plist (c->eperm = right-hand side).
int64_t run_pcg_pre(mdg_ctx* c, double tol_debye, int64_t max_iter, double* last_rms);
// The same over several domains (one stream) with halo exchange and summed
// CG scalars through comm (NULL: one domain).
int64_t run_pcg_multi(std::vector<mdg_ctx*> doms, PcgComm* comm, double tol_debye,
                      int64_t max_iter, double* last_rms);
void pcg_graph_forget(const void* owner);
// domain groups (group.cu)
PcgComm* group_comm(mdg_group* g);
std::vector<mdg_ctx*> group_domains(mdg_group* g);
bool group_is_nccl(mdg_group* g);
void group_refresh(mdg_group* g);
void group_sum_host(mdg_group* g, double* v, int nv);
// debug builds (-DMDG_DEBUG): device-assert every row's count <= cap, every
// neighbour index in [0, n_all) and != the row's site, ascending when sorted
// (debug.cu); a no-op in the product build
void debug_check_rows(mdg_ctx* c, const char* what, const int32_t* nbr, const int32_t* cnt,
                      int32_t cap, int64_t rows, int64_t n_all, bool sorted);
// device spatial re-sort of every per-site array (resort.cu); invalidates lists
// rep (device, may be NULL): per site, the sorted index of its molecule's
// representative -> molecule-keyed order (also kept by later re-sorts)
void resort_sites(mdg_ctx* c, const int32_t* rep = nullptr);
bool mol_order_fits(const mdg_ctx* c);
// vdW sites from the positions (Halgren reduction or copy), after new positions
void refresh_vsites(mdg_ctx* c);
void run_reduce_sites(mdg_ctx* c);
// polarization forces at c->mu (polforce.cu); results slots 70 (pair
// energy), 71..79 (virial); accumulate adds to c->force / c->torque
void run_polar_force(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                     double electric, int exclude, bool accumulate);
void run_polar_force_pruned(mdg_ctx* c, double alpha, double thole_a, double electric,
                            int exclude, bool accumulate);
// local frames: mp <- R mploc (every entry point that reads multipoles) and
// torque -> forces on the frame atoms (after the torque kernels)
void rotate_multipoles(mdg_ctx* c);
void frame_torques_to_forces(mdg_ctx* c);
// smooth PME reciprocal space for point charges (pme.cu): adds forces to
// c->force; results 80 (recip), 81-86 (virial), 87 (self), 88-97 (excluded)
void run_pme(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order, double electric,
             bool exclude);
void pme_free(mdg_ctx* c);
// list staleness (nlist.cu): positions snapshot at build / import; host check
// of the fetched results (throws MDG_CONTRACT)
void list_snapshot(mdg_ctx* c, int list_id);
void check_lists_fresh(const mdg_ctx* c);
// smooth PME for permanent multipoles (q, mu, Theta): adds forces and torques;
// results 80 (recip), 88 (excluded pairs), 98 (recip from the gathered
// potentials), 104-106 (sums of q^2, |mu|^2, Q:Q for the self energy)
// ind != NULL: the permanent + induced set (the polarization forces' pass:
// forces of the whole set, torques on the permanent multipoles, no energies;
// excluded pairs keep their induced-induced part); forces == false: energies only
void run_pme_mpole(mdg_ctx* c, double alpha, int k1, int k2, int k3, int order,
                   double electric, bool exclude, const double4* ind = nullptr,
                   bool forces = true);
// reciprocal + self Ewald field (c->pol_recip): mode 0 adds the permanent
// multipoles' field (and removes the excluded pairs' erf part) to out; mode 1
// adds v's dipole field to out; mode 2 (PCG) subtracts it from out and writes
// the block partials of v.out
void pme_field(mdg_ctx* c, int mode, const double4* v, double4* out);
// the same over the domains of a group (replicated grid summed through comm;
// comm == NULL: one domain). mode 0: v = none, out = eperm; 1: v = mu,
// out = cg_q; 2: v = cg_p, out = cg_q. ind: the permanent + induced set (mu).
void pme_field_multi(const std::vector<mdg_ctx*>& doms, PcgComm* comm, int mode);
void run_pme_mpole_multi(const std::vector<mdg_ctx*>& doms, PcgComm* comm, double alpha, int k1,
                         int k2, int k3, int order, double electric, bool exclude, bool ind,
                         bool forces);
// MD (md.cu): bonded forces added to c->force (results 100 bonds, 101
// angles), velocity-Verlet half kick / drift, kinetic energy (result 102)
void run_bonded(mdg_ctx* c);
void run_bonded(mdg_ctx* c, double4* out);  // adds into out
void run_kick(mdg_ctx* c, double half_dt);
void run_kick(mdg_ctx* c, double half_dt, const double4* force);
// Langevin O step: v = c1 v + sqrt(1 - c1^2) sqrt(kT/m) xi (kt in kcal/mol)
void run_ostep(mdg_ctx* c, double c1, double kt, uint64_t seed, uint64_t counter);
void run_drift(mdg_ctx* c, double dt);
void run_kinetic(mdg_ctx* c);


// permutation helpers (device kernels)
void scatter_sorted_scalar(mdg_ctx* c, const double* d_src, double* d_dst_sorted);
void gather_vec_to_caller(mdg_ctx* c, const double4* sorted, double* d_dst_soa);
void scatter_vec_from_caller(mdg_ctx* c, const double* d_src_soa, double4* sorted);
void zero_vec(mdg_ctx* c, double4* v);
void pack_system(mdg_ctx* c);
void set_vdw_types(mdg_ctx* c, const std::vector<int32_t>& rep);
double4* vec_by_id(mdg_ctx* c, int vec_id);
void vec_pack(mdg_ctx* c, int vec_id, const int32_t* d_sites, int64_t count, double* d_out);
void vec_unpack(mdg_ctx* c, int vec_id, const int32_t* d_sites, int64_t count,
                const double* d_in);
void pack_positions(mdg_ctx* c, int64_t count = -1);
// pos.w / vsite.w <- mol (after a topology upload)
void set_groups(mdg_ctx* c);
// device check of staged positions against the box; first bad caller index or -1
int64_t check_box_staged(mdg_ctx* c, int64_t count = -1);
void polar_energy(mdg_ctx* c, double electric, int slot);

}  // namespace mdg
