/*
 * mdg.h -- C ABI of the B200-native (sm_100a) FP64 real-space pair engine.
 *
 * Drop-in boundary for the reference `mdvec` hot path (/root/reference/proj).
 * The reference has no FFI; its boundary is the C++ header API. Each entry
 * point below names the reference interface it replaces (file:line). A C++
 * wrapper that keeps the reference signatures and exception types lives in
 * include/mdvec_gpu.hpp; the Python mirror in paper_1906_01211_b200/mdvec.py.
 *
 * Conventions
 *  - Every function returns an int status: 0 OK, 1 CONTRACT (reference
 *    ContractViolation), 2 CAPACITY (CapacityError), 3 SINGULARITY,
 *    4 CONVERGENCE (ConvergenceError), 5 CUDA, 6 COMM. mdg_last_error()
 *    returns a thread-local message for the last failure.
 *  - Host arrays are in the caller's site order (the reference's). The
 *    context keeps a spatially sorted copy on the device and permutes at the
 *    boundary; results are bit-for-bit independent of the caller's order only
 *    up to FP summation order.
 *  - Outputs are OVERWRITTEN (reference `out.reset()`, e.g.
 *    proj/src/kernels_scalar.cpp:13). Results are ready on return
 *    (synchronous), as in the reference.
 *  - Per-site vectors (forces, fields, dipoles, torques) are SoA
 *    (x[], y[], z[]) like ForceAccumulator / FieldArrays /
 *    PolarizationState (proj/include/mdvec/kernels.hpp:21-34,
 *    polar.hpp:74-84, system.hpp:36-42). Any output pointer may be NULL.
 *  - virial9: row-major W_ab = sum over pairs of d_a F_b, d = r_i - r_j
 *    (minimum image), F = force on i from j. Not in the reference.
 *  - A context is single-stream and not thread-safe; use one per thread
 *    (reference SPEC: concurrent calls on disjoint outputs).
 */
#ifndef MDG_H
#define MDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDG_OK 0
#define MDG_CONTRACT 1
#define MDG_CAPACITY 2
#define MDG_SINGULARITY 3
#define MDG_CONVERGENCE 4
#define MDG_CUDA 5
#define MDG_COMM 6

#define MDG_MAX_LISTS 4
#define MDG_SITES_ATOMIC 0 /* list over atomic positions */
#define MDG_SITES_VDW 1    /* list over Halgren-reduced vdW sites */

#define MDG_MAX_NEIGHBORS 2560 /* proj/include/mdvec/common.hpp:10 (half list) */

typedef struct mdg_ctx mdg_ctx;

const char* mdg_last_error(void);
int mdg_version(void);

/* ---- context ------------------------------------------------------------ */
/* One device, one stream, capacity fixed at create time (the reference's
 * preallocation contract, proj/tests/test_layout.cpp:215-237).
 * max_pairs_per_atom bounds the FULL (both-direction) list per site; 0 picks
 * 2 * MDG_MAX_NEIGHBORS. */
int mdg_ctx_create(mdg_ctx** out, int device, int64_t n_capacity, int32_t max_pairs_per_atom);
int mdg_ctx_destroy(mdg_ctx* ctx);
int mdg_ctx_synchronize(mdg_ctx* ctx);
/* cudaStream_t of the context, for callers that time on it. */
void* mdg_ctx_stream(mdg_ctx* ctx);

/* ---- system ------------------------------------------------------------- */
/* Replaces ParticleSystem (proj/include/mdvec/system.hpp:12-25); validation
 * as ParticleSystem::validate (proj/src/system.cpp:9-28). Sets the site
 * order (spatial sort) used until the next mdg_system_upload. */
int mdg_system_upload(mdg_ctx* ctx, int64_t n, double lx, double ly, double lz,
                      const double* x, const double* y, const double* z, const double* charge,
                      const double* lj_sigma, const double* lj_epsilon, const double* hal_r0,
                      const double* hal_epsilon, const double* polarizability);
/* New coordinates for the same sites (one MD step's input). Lists are kept. */
int mdg_positions_upload(mdg_ctx* ctx, const double* x, const double* y, const double* z);
/* Domain contexts: the owned sites' coordinates only (n_own entries, the
 * owned part of the caller order); the halo follows from
 * mdg_group_exchange(g, MDG_VEC_POS). */
int mdg_positions_upload_owned(mdg_ctx* ctx, const double* x, const double* y, const double* z);
/* Topology (no reference counterpart): molecule ids (exclusion groups; NULL =
 * every site its own group) and the Halgren reduction parent/factor (NULL =
 * no reduction: vdW sites = atoms). With molecule ids, a one-domain context
 * re-orders its resident sites so each molecule's sites are consecutive
 * (the molecule tiles of the Halgren / PCG cluster kernels; MDG_MOL_ORDER=0
 * keeps the site order): neighbour lists built before must be built again.
 * The caller-order interface is unaffected. */
int mdg_topology_upload(mdg_ctx* ctx, const int32_t* molecule, const int32_t* hred_parent,
                        const double* hred_factor);
/* Permanent multipoles (no reference counterpart): dipole[3n] (x,y,z per
 * site), quadrupole[6n] traceless (xx,xy,xz,yy,yz,zz per site, Tinker's
 * convention: Theta/3). NULL zeroes the term. Charges come from the system. */
int mdg_multipoles_upload(mdg_ctx* ctx, const double* dipole, const double* quadrupole);
/* Local multipole frames (Tinker conventions): per site
 * frame_type 0 = none (multipoles global), 1 = z-then-x, 2 = bisector, with
 * zatom / xatom the caller-order frame atoms (same molecule). dipole[3n] and
 * quadrupole[6n] are then given in the local frame; every multipole entry
 * point rotates them to the global frame at the current positions, and the
 * multipole / polarization torques are turned into forces on the frame atoms
 * (included in the returned forces; torques are still reported). NULL
 * frame_type removes the frames. */
int mdg_frames_upload(mdg_ctx* ctx, const int32_t* frame_type, const int32_t* zatom,
                      const int32_t* xatom, const double* dipole, const double* quadrupole);

/* ---- neighbour lists ---------------------------------------------------- */
/* Replaces build_cell_grid + build_neighbor_table
 * (proj/include/mdvec/neighbors.hpp:43-50, proj/src/neighbors_vec.cpp:8-94).
 * Contract checks as proj/src/neighbors.cpp:10-17 (cutoff > 0, <= L/2).
 * The device list holds every pair (both directions) within list_cutoff. */
int mdg_nlist_build(mdg_ctx* ctx, int list_id, double list_cutoff, int sites);
/* half_pairs = number of (i<j) pairs; padded_slots = reference-layout total. */
int mdg_nlist_size(mdg_ctx* ctx, int list_id, int64_t* half_pairs, int64_t* padded_slots);
/* Reference NeighborTable layout (proj/include/mdvec/neighbors.hpp:22-41):
 * pairs stored on the lower site index, segments padded to 16 with the last
 * neighbour as sentinel, so table_pairs() (neighbors.cpp:59-72) applies.
 * Neighbours within a segment are ascending. */
int mdg_nlist_export(mdg_ctx* ctx, int list_id, uint32_t* nnvlst, uint32_t* nvloop8,
                     uint32_t* nvloop16, uint64_t* offset, int32_t* indices,
                     int64_t indices_cap);
/* Feeds a reference-layout table (e.g. one built by the reference, or
 * exclusion-filtered) so a kernel runs on exactly that pair set. */
int mdg_nlist_import(mdg_ctx* ctx, int list_id, double list_cutoff, int sites,
                     const uint32_t* nnvlst, const uint64_t* offset, const int32_t* indices);

/* ---- nonpolar kernels ----------------------------------------------------
 * exclude != 0 skips pairs of one molecule. electric multiplies Coulomb
 * terms (reference: 1.0; SI-ish MD: 332.063713). On a list over vdW sites
 * the forces are chain-ruled back onto atoms. */
/* lj_forces_{scalar,vectorized}, proj/include/mdvec/kernels.hpp:101-105 */
int mdg_lj_forces(mdg_ctx* ctx, int list_id, double cutoff, int shift, int exclude,
                  double* fx, double* fy, double* fz, double* energy, double* virial9);
/* ewald_real_forces_*, proj/include/mdvec/kernels.hpp:107-114 */
int mdg_ewald_real_forces(mdg_ctx* ctx, int list_id, double alpha, double cutoff,
                          double electric, int exclude, double* fx, double* fy, double* fz,
                          double* energy, double* virial9);
/* halgren_forces_*, proj/include/mdvec/polar.hpp:86-91 */
int mdg_halgren_forces(mdg_ctx* ctx, int list_id, double cutoff, double delta, double gamma,
                       int exclude, double* fx, double* fy, double* fz, double* energy,
                       double* virial9);

/* ---- polarization ------------------------------------------------------- */
/* dipole_field_matvec_* (proj/include/mdvec/polar.hpp:95-104) generalised
 * to real-space Ewald: rr3 = B1 - (1-l3)/r^3, rr5 = B2 - 3(1-l5)/r^5. At
 * alpha = 0 this is the reference Thole-only T. All list pairs (u-scale 1). */
int mdg_tmatvec(mdg_ctx* ctx, int list_id, double alpha, double cutoff, double thole_a,
                const double* mux, const double* muy, const double* muz, double* ex,
                double* ey, double* ez);
/* permanent_field_* (proj/include/mdvec/polar.hpp:107-112) generalised to
 * q + mu + Theta and real-space Ewald (Thole l3/l5/l7). At alpha = 0 with no
 * multipoles uploaded this is the reference charge-only field. */
int mdg_perm_field(mdg_ctx* ctx, int list_id, double alpha, double cutoff, double thole_a,
                   int exclude, double* ex, double* ey, double* ez);
/* jacobi_polarization_solve (proj/include/mdvec/polar.hpp:115-118), same
 * max-norm stopping rule, on the device. */
int mdg_polar_solve_jacobi(mdg_ctx* ctx, int list_id, double cutoff, double thole_a, double tol,
                           int64_t max_iter, double* mux, double* muy, double* muz,
                           int64_t* iters, double* last_residual);
/* Diagonal-preconditioned CG for (alpha^-1 - T) mu = E_perm (no reference
 * counterpart; the reference solver is Jacobi). mu0 = alpha E. Stops when
 * sqrt(sum|dmu|^2/n) * 4.80321 < tol_debye. E_perm from mdg_perm_field with
 * the same alpha/cutoff/thole_a and exclude_perm. */
int mdg_polar_solve_pcg(mdg_ctx* ctx, int list_id, double alpha, double cutoff, double thole_a,
                        int exclude_perm, double tol_debye, int64_t max_iter, double* mux,
                        double* muy, double* muz, int64_t* iters, double* last_rms_debye);

/* ---- permanent multipoles (empole1 analogue, no reference counterpart) ---- */
/* Real-space Ewald q/mu/Theta energy, translational forces, torques (global
 * frame) and pair virial. */
int mdg_mpole_forces(mdg_ctx* ctx, int list_id, double alpha, double cutoff, double electric,
                     int exclude, double* fx, double* fy, double* fz, double* tx, double* ty,
                     double* tz, double* energy, double* virial9);

/* ---- polarization forces (epolar1 analogue) -------------- */
/* Forces, torques on the permanent multipoles and pair virial of the
 * polarization energy at fixed induced dipoles mu (caller order, e*A; NULL =
 * the context's dipoles from its last solve): F = -dE/dr of
 * E = 1/2 mu.a^-1.mu - 1/2 mu.T.mu - mu.E_perm with the same Ewald + Thole
 * T and field as mdg_polar_solve_pcg / mdg_perm_field (exact forces at the
 * converged solution). pair_energy = the mu-dependent pair part of E
 * (E = pair_energy + 1/2 sum mu^2/alpha). */
int mdg_polar_forces(mdg_ctx* ctx, int list_id, double alpha, double cutoff, double thole_a,
                     double electric, int exclude, const double* mux, const double* muy,
                     const double* muz, double* fx, double* fy, double* fz, double* tx,
                     double* ty, double* tz, double* pair_energy, double* virial9);

/* ---- reciprocal-space Ewald -------------------------------- */
/* Smooth PME for the point charges on a k1 x k2 x k3 grid with order-`order`
 * B-splines (cuFFT): forces (overwritten), energies3 = (reciprocal, self
 * -a/sqrt(pi) sum q^2, excluded-pair correction -sum q_i q_j erf(a r)/r over
 * same-molecule pairs when exclude != 0), virial9 = reciprocal + excluded
 * (strain derivative, the pair-virial convention). With mdg_ewald_real_forces
 * at the same alpha the four terms are the full Ewald sum. Single domain. */
int mdg_ewald_recip(mdg_ctx* ctx, double alpha, int k1, int k2, int k3, int order,
                    double electric, int exclude, double* fx, double* fy, double* fz,
                    double* energies3, double* virial9);

/* Smooth PME for the permanent multipoles (charge, dipole, quadrupole;
 * 8(f)#3): site operator q + mu.grad + Q:grad grad spread with B-splines of
 * order 5..10 and their derivatives, cuFFT, potential derivatives to third
 * order gathered per site. forces and torques (overwritten, global frame;
 * with local frames the torques are NOT turned into frame forces here),
 * energies3 = (reciprocal, self -a/sqrt(pi) sum [q^2 + 2a^2|mu|^2/3 +
 * 8a^4 Q:Q/5], excluded-pair correction: minus the erf(a r)/r-kernel
 * interaction of same-molecule pairs when exclude != 0). With
 * mdg_mpole_forces at the same alpha the four terms are the full multipole
 * Ewald sum. Single domain. */
int mdg_ewald_recip_mpole(mdg_ctx* ctx, double alpha, int k1, int k2, int k3, int order,
                          double electric, int exclude, double* fx, double* fy, double* fz,
                          double* tx, double* ty, double* tz, double* energies3);

/* Reciprocal-space Ewald in the AMOEBA-style step and mdg_polar_solve_pcg
 * (8(f)#3), single domain: with a k1 x k2 x k3 grid and B-spline order 5..10
 * set, the permanent field (PCG right-hand side) gains the multipoles'
 * reciprocal field, the Ewald self field 4a^3/(3 sqrt(pi)) mu and (with the
 * call's exclusions) minus the erf-kernel field of same-molecule partners;
 * the PCG operator gains the reciprocal + self field of the dipoles (one
 * smooth-PME pass per iteration); the step's multipole term gains
 * mdg_ewald_recip_mpole's energy, forces and torques. The polarization
 * energy -1/2 mu.E_perm is then the full Ewald one. With
 * MDG_TERM_POLAR_FORCE (and MDG_TERM_MPOLE) the reciprocal-space forces and
 * torques of multipoles + polarization come from one pass over the
 * permanent + induced set after the solve (torques on the permanent
 * multipoles only). k1 = 0 switches it off (default). */
int mdg_set_ewald_recip(mdg_ctx* ctx, int k1, int k2, int k3, int order);

/* ---- fused steps (device-resident; the bench's hot path) ----------------- */
typedef struct {
  double cutoff;    /* LJ and Ewald cutoff (A) */
  double alpha;     /* Ewald alpha (1/A) */
  double electric;  /* Coulomb constant */
  int shift;        /* LJ shift */
  int exclude;      /* intramolecular exclusions */
} mdg_charmm_params;

/* Config-0 step: fused LJ + real-space Ewald charge energy, forces, virial
 * over list list_id. Results stay on the device (mdg_fetch_forces). */
int mdg_charmm_step(mdg_ctx* ctx, int list_id, const mdg_charmm_params* p);

typedef struct {
  double vdw_cutoff, delta, gamma;          /* Halgren */
  double elec_cutoff, alpha, electric;      /* multipoles, field, T */
  double thole_a, tol_debye;
  int64_t max_iter;
  int exclude;                              /* 1-2/1-3 (intramolecular) scale 0 */
  int terms;                                /* MDG_TERM_* bits (0 = VDW|MPOLE|POLAR) */
} mdg_amoeba_params;

#define MDG_TERM_VDW 1
#define MDG_TERM_MPOLE 2
#define MDG_TERM_POLAR 4
/* with POLAR: add the polarization forces/torques/virial at the converged
 * dipoles (8(f)#1) to the step's results */
#define MDG_TERM_POLAR_FORCE 8

/* Config-1..4 step: Halgren vdW (list vdw_list, reduced sites) + permanent
 * multipoles + permanent field + PCG induced dipoles (list elec_list).
 * Results stay on the device. */
int mdg_amoeba_step(mdg_ctx* ctx, int vdw_list, int elec_list, const mdg_amoeba_params* p);

/* ---- MD time loop ----------------------------------------- */
/* Harmonic bonded terms for flexible molecules (caller-order site ids):
 * bond energy kb (r - r0)^2, angle energy ka (theta - theta0)^2 (radians,
 * angles[3k+1] the vertex). Replaces any previous set. */
int mdg_bonded_upload(mdg_ctx* ctx, int64_t nbonds, const int32_t* bonds, const double* kb,
                      const double* r0, int64_t nangles, const int32_t* angles,
                      const double* ka, const double* theta0);
/* Bonded forces alone (overwrite) and energies2 = (bonds, angles). */
int mdg_bonded_forces(mdg_ctx* ctx, double* fx, double* fy, double* fz, double* energies2);
/* Masses (amu; NULL keeps the previous ones) and velocities (A/fs). */
int mdg_velocities_upload(mdg_ctx* ctx, const double* mass, const double* vx, const double* vy,
                          const double* vz);
int mdg_velocities_fetch(mdg_ctx* ctx, double* vx, double* vy, double* vz);
int mdg_positions_fetch(mdg_ctx* ctx, double* x, double* y, double* z);

typedef struct {
  int model;             /* 0 CHARMM-style (charmm params), 1 AMOEBA-style */
  int64_t nsteps;
  double dt_fs;
  int rebuild_every;     /* neighbour lists rebuilt every this many steps */
  int elec_list, vdw_list;              /* list ids (vdw_list: AMOEBA only) */
  double elec_list_cutoff, vdw_list_cutoff;
  int bonded;            /* add the uploaded bonded terms */
  /* integrator (zero-initialised fields keep velocity Verlet) */
  int integrator;        /* MDG_INTEGRATOR_VERLET or MDG_INTEGRATOR_BAOAB_RESPA */
  int inner_steps;       /* BAOAB-RESPA: bonded sub-steps per outer step (>= 1) */
  double friction_ps;    /* BAOAB-RESPA: Langevin friction (1/ps); 0 = NVE RESPA */
  double temperature_k;  /* BAOAB-RESPA: bath temperature (K) */
  uint64_t seed;         /* BAOAB-RESPA: noise stream (counter-based, per caller site) */
  int predictor;         /* AMOEBA: PCG start, MDG_PREDICT_NONE (alpha E) or _ASPC */
} mdg_md_params;

/* ASPC (Kolafa 2004, k = 4): the PCG of each step starts from the dipoles
 * extrapolated from the last 6 converged ones (the paper's "Beeman/ASPC"
 * production setup); the solve still runs to its tolerance. The history is
 * kept within one mdg_md_run call and cleared by a re-sort. */
#define MDG_PREDICT_NONE 0
#define MDG_PREDICT_ASPC 1

#define MDG_INTEGRATOR_VERLET 0
#define MDG_INTEGRATOR_BAOAB_RESPA 1

/* nsteps on the device (single domain).
 * Velocity Verlet: kick, drift (positions wrapped into the box), lists
 * rebuilt on schedule, forces of the selected model (+ bonded), kick.
 * BAOAB-RESPA (the multi-timestep Langevin scheme of the paper's Rel2,
 * /root/reference/PAPER.md:782-783, two levels): the nonbonded model is the
 * outer level at dt_fs, the bonded terms the inner level at
 * dt_fs / inner_steps:
 *   B_out(dt/2) [ B_in(h/2) A(h/2) O(h) A(h/2) F_in B_in(h/2) ] x inner_steps
 *   F_out B_out(dt/2)
 * with O: v = c1 v + sqrt((1 - c1^2) kT / m) xi, c1 = exp(-friction h), xi
 * a SplitMix64/Box-Muller deviate of (seed, inner-step counter, caller site,
 * component). ekin / epot (kcal/mol, NULL to skip) receive each step's
 * kinetic / potential energy; the AMOEBA model needs MDG_TERM_POLAR_FORCE
 * with polarization for conservative dynamics. */
int mdg_md_run(mdg_ctx* ctx, const mdg_md_params* p, const mdg_charmm_params* charmm,
               const mdg_amoeba_params* amoeba, double* ekin, double* epot);
/* List rebuilds done by mdg_md_run so far (all calls): rebuild_every is the
 * longest interval; a rebuild comes earlier when the device has seen a site
 * move 0.6 x the motion its list tolerates (half of list cutoff minus the
 * kernel's cutoff and row buffer) since the build. A list walked past that
 * tolerance would miss pairs: result reads then fail with MDG_CONTRACT. */
int mdg_md_rebuild_count(mdg_ctx* ctx, int64_t* count);

/* Spatial re-sort on the device: the sites are re-keyed by their current
 * ~2 A Morton cells and every per-site array is permuted (index arrays
 * remapped), restoring the gathers' locality after the sites have moved.
 * mdg_md_run does it at every 20th list rebuild, counted across calls
 * (MDG_RESORT=k: every k-th; 0 disables). The
 * caller-order interface is unchanged; neighbour lists are invalidated
 * (rebuild them). Single domain only. */
int mdg_resort(mdg_ctx* ctx);

/* Results of the last step / kernel, copied to host (caller order).
 * energies[4] = {vdw, coulomb or multipole, polarization (0 here), unused}. */
int mdg_fetch_forces(mdg_ctx* ctx, double* fx, double* fy, double* fz);
/* Register page-locked caller arrays (mdg_host_alloc) as the force output:
 * every later charmm/amoeba step queues the DMA of its final forces into
 * them as soon as they are complete (for the AMOEBA step without
 * polarization forces or frames: while the PCG still runs), and an
 * mdg_fetch_forces with the same pointers called right after the step only
 * waits for it. The arrays are written asynchronously by each step: read
 * them after mdg_fetch_forces / mdg_ctx_synchronize. NULLs unregister; a new
 * system upload unregisters. No counterpart in the reference (its kernels
 * write caller arrays directly, proj/include/mdvec/kernels.hpp ForceResult). */
int mdg_set_force_output(mdg_ctx* ctx, double* fx, double* fy, double* fz);
int mdg_fetch_torques(mdg_ctx* ctx, double* tx, double* ty, double* tz);
int mdg_fetch_dipoles(mdg_ctx* ctx, double* mux, double* muy, double* muz);
/* Permanent field (PCG right-hand side) of the last step / PCG solve. */
int mdg_fetch_perm_field(mdg_ctx* ctx, double* ex, double* ey, double* ez);
int mdg_fetch_energies(mdg_ctx* ctx, double* energies4, double* virial9, int64_t* pcg_iters,
                       double* pcg_rms);

/* ---- spatial domain decomposition (one context per GPU / rank) ----------- */
/* Device vectors addressable by the halo exchange. */
#define MDG_VEC_POS 0    /* x, y, z (charges stay) */
#define MDG_VEC_MU 1     /* induced dipoles */
#define MDG_VEC_P 2      /* PCG search direction */
#define MDG_VEC_FORCE 3
#define MDG_VEC_TORQUE 4
#define MDG_VEC_EPERM 5

/* Like mdg_system_upload, but only the first n_owned caller sites are owned
 * by this context (their rows are computed: forces, fields, dipoles); the
 * rest are the halo (inputs only). n_global counts every site of every
 * domain (PCG RMS normalisation). n_owned == n reproduces mdg_system_upload. */
int mdg_system_upload_owned(mdg_ctx* ctx, int64_t n, int64_t n_owned, int64_t n_global,
                            double lx, double ly, double lz, const double* x, const double* y,
                            const double* z, const double* charge, const double* lj_sigma,
                            const double* lj_epsilon, const double* hal_r0,
                            const double* hal_epsilon, const double* polarizability);
/* ---- domain groups: the decomposed system's runtime (group.cu) ------------
 * A group is the set of domain contexts of one spatially decomposed system
 * (each created with mdg_system_upload_owned: owned sites first, then the
 * halo). The group refreshes halos and, inside the PCG solve, exchanges the
 * search direction and sums the CG scalars over all domains on the device:
 * no host round trip per iteration. No reference counterpart (the reference
 * is single-process; Tinker-HP's spatial
 * decomposition). */
typedef struct mdg_group mdg_group;
#define MDG_GROUP_LOCAL 0 /* several domains in this process, one device */
#define MDG_GROUP_NCCL 1  /* one domain per process (rank), NCCL over NVLink */

/* NCCL unique id (128 bytes): rank 0 makes it, every rank passes it to
 * mdg_group_create_nccl (broadcast out of band, e.g. torch.distributed). */
int mdg_nccl_unique_id(void* id128);
/* LOCAL group of n domain contexts on one device. They share the first
 * context's stream while grouped (restored by mdg_group_destroy). n_global
 * counts the sites of the whole system (PCG RMS normalisation). */
int mdg_group_create_local(mdg_group** out, int n, mdg_ctx** ctxs, int64_t n_global);
/* NCCL group: this process's domain context as rank `rank` of `size`. */
int mdg_group_create_nccl(mdg_group** out, mdg_ctx* ctx, int rank, int size, const void* id128,
                          int64_t n_global);
int mdg_group_destroy(mdg_group* g);
/* Interior/halo overlap inside the PCG: each iteration's halo refresh of the
 * search direction runs on the group's communication stream while the
 * mat-vec of the sites whose pruned rows hold no halo site runs on the
 * domains' stream; the boundary sites follow once the halo is in. Default:
 * on for NCCL groups, off for LOCAL ones (one device: the pull kernel is too
 * small to hide anything); the environment variable MDG_DD_OVERLAP=0/1 sets
 * the default. */
int mdg_group_set_overlap(mdg_group* g, int on);
/* mdg_ctx_destroy of a grouped context fails with MDG_CONTRACT: destroy the
 * group first. */
/* LOCAL halo of domain `domain`: for each of its n_halo halo sites (caller-
 * order local index halo_site[k]) the owning domain src_domain[k] and the
 * site's caller-order local index there, src_site[k]. */
int mdg_group_set_halo_local(mdg_group* g, int domain, int64_t n_halo, const int32_t* halo_site,
                             const int32_t* src_domain, const int32_t* src_site);
/* NCCL halo: per peer rank (peers[p]), send_counts[p] owned sites it needs
 * and recv_counts[p] halo sites it sends, as caller-order local indices
 * concatenated per peer, in the order both sides agree on (global id). */
int mdg_group_set_halo_nccl(mdg_group* g, int npeers, const int32_t* peers,
                            const int64_t* send_counts, const int32_t* send_sites,
                            const int64_t* recv_counts, const int32_t* recv_sites);
/* Refresh the halo entries of vec_id (MDG_VEC_*) in every local domain from
 * their owners (POS also refreshes the Halgren-reduced halo sites). Returns
 * after completion. */
int mdg_group_exchange(mdg_group* g, int vec_id);
/* Snapshot every domain's owned positions as the plan's reference, and the
 * largest minimum-image displacement of any owned site since (max over all
 * domains / ranks): the halo misses no pair while it stays below half the
 * halo margin (halo width - list cutoff - intramolecular extent). */
int mdg_group_set_reference(mdg_group* g);
int mdg_group_max_displacement(mdg_group* g, double* out);
/* Sum result slots [slot, slot + nv) over all domains / ranks, in place, on
 * the device (stream-ordered; nv <= 32). */
int mdg_group_allreduce_results(mdg_group* g, int slot, int nv);
/* mdg_amoeba_step for every local domain: per domain Halgren, field + T
 * tensors and multipoles; one PCG over all domains (halo of the search
 * direction and summed CG scalars every iteration, on the device); then the
 * polarization forces after a halo refresh of the dipoles. */
int mdg_group_amoeba_step(mdg_group* g, int vdw_list, int elec_list, const mdg_amoeba_params* p);
int mdg_group_charmm_step(mdg_group* g, int list_id, const mdg_charmm_params* p);
/* Energies and virial summed over all domains (and ranks); PCG record. */
int mdg_group_fetch_energies(mdg_group* g, double* energies4, double* virial9,
                             int64_t* pcg_iters, double* pcg_rms);
/* Pair-sum mode of the Halgren and multipole kernels. Default (0): each
 * owned-owned pair is evaluated once (Newton's third law, as the reference's
 * half lists do) and the partner's force/torque is added with FP64 atomics,
 * so the last bits of forces can vary run to run. 1: every site sums its
 * full row in a fixed order (twice the pair arithmetic, bitwise
 * reproducible). The environment variable MDG_DETERMINISTIC sets the
 * default of new contexts. Energies and virials are reproducible in both. */
int mdg_set_deterministic(mdg_ctx* ctx, int on);
/* AMOEBA step scheduling. Default (1): Halgren and the multipoles run on a
 * low-priority second stream beside the field -> PCG chain; 0: one stream
 * (kernel-by-kernel profiling). MDG_OVERLAP=0 sets the default of new
 * contexts. Results are the same either way. */
int mdg_set_overlap(mdg_ctx* ctx, int on);
/* PCG on site clusters (default 0; MDG_CLUSTER_MATVEC=1 sets the default of
 * new contexts): per cluster of 3 consecutive sites (a water molecule in the
 * molecule-keyed site order) the union of the sites' buffered rows, the field
 * pass writing each site's pair tensors into the union's slots, and a PCG
 * mat-vec that streams those with one gather of j per union entry (bulk
 * asynchronous copies into shared memory). Measured on config 4 at parity
 * with the per-site rows in the mat-vec and slower in the field pass
 * (DESIGN.md section 4). Applies only to buffered cut rows without an
 * overlapped domain exchange. The dipoles agree to rounding either way. */
int mdg_set_cluster_matvec(mdg_ctx* ctx, int on);
/* Halgren on site clusters (default 1; MDG_CLUSTER_HALGREN=0 sets the
 * default of new contexts): per cluster of 3 consecutive sites (a water
 * molecule in the molecule-keyed order) the union of the sites' buffered
 * half rows, walked once with a lane per union entry -- j's record gathered
 * and its partner force added once for the three sites. The per-site half
 * rows otherwise (in deterministic mode and for unbuffered rows). The same
 * pairs either way. */
int mdg_set_cluster_halgren(mdg_ctx* ctx, int on);
/* Gather 3 doubles per listed caller-order site of vec_id into out[3*count]
 * (x,y,z interleaved) / scatter them back. Host buffers. */
int mdg_vec_pack(mdg_ctx* ctx, int vec_id, const int32_t* sites, int64_t count, double* out);
int mdg_vec_unpack(mdg_ctx* ctx, int vec_id, const int32_t* sites, int64_t count,
                   const double* in);
/* Same with device-resident index and data buffers (e.g. NCCL send/recv
 * buffers); ordered on the context stream, returns after completion. */
int mdg_vec_pack_dev(mdg_ctx* ctx, int vec_id, const int32_t* d_sites, int64_t count,
                     double* d_out);
int mdg_vec_unpack_dev(mdg_ctx* ctx, int vec_id, const int32_t* d_sites, int64_t count,
                       const double* d_in);

/* ---- instrumentation ---------------------------------------------------- */
/* Fault injection, the analogue of the reference bench's
 * debug_perturb_vectorized (proj/include/mdvec/bench.hpp:42-44,
 * proj/src/bench.cpp:244-255): delta is added to the x force of the first
 * site returned by mdg_fetch_forces and to energies[0] of
 * mdg_fetch_energies, so a parity check downstream must flag the results.
 * 0 (default) disables it. */
int mdg_set_debug_perturb(mdg_ctx* ctx, double delta);
/* CUDA events on the context stream: start records, stop records, waits and
 * returns the elapsed device milliseconds. */
int mdg_timer_start(mdg_ctx* ctx);
int mdg_timer_stop(mdg_ctx* ctx, double* ms);
/* Counts kernel launches issued by this context since creation/reset. */
int64_t mdg_launch_count(mdg_ctx* ctx);
/* When enabled, every launch is bracketed by CUDA events on the context
 * stream and accumulated per kernel name. */
int mdg_profile_enable(mdg_ctx* ctx, int enable);
int mdg_profile_reset(mdg_ctx* ctx);
/* Writes "name count total_ms\n" lines into buf (NUL terminated). */
int mdg_profile_report(mdg_ctx* ctx, char* buf, int64_t buf_len);

/* Page-locked host buffers: per-step inputs/outputs that live here skip the
 * staging copy (positions are DMA'd straight from them, results straight
 * into them). Any pointer works with every call; pinned ones are faster. */
int mdg_host_alloc(void** ptr, int64_t bytes);
int mdg_host_free(void* ptr);

/* FP64 DFMA-chain peak probe on `device` (TFLOP/s, best of 5). */
int mdg_probe_fp64_peak(int device, double* tflops);
/* The pair kernels' device erfc (exp(-x^2) * erfcx polynomial, common.cuh)
 * evaluated at n host points: accuracy check against a host erfc. */
int mdg_probe_erfc(int device, const double* x, int64_t n, double* out);
/* Directed (both-direction) pairs of list_id within cutoff (minus excluded
 * pairs when exclude != 0) and total list slots: roofline numerators. */
int mdg_nlist_count_within(mdg_ctx* ctx, int list_id, double cutoff, int exclude,
                           int64_t* directed_pairs, int64_t* list_slots);

/* ---- synthetic water fixtures (BASELINE.json configs) -------------------- */
/* n_mol rigid 3-site waters (O,H,H per molecule, molecule-major) in a cubic
 * box of edge L, jittered lattice + uniform random orientation, std::
 * mt19937_64(seed). Outputs (length 3*n_mol unless noted):
 *   x,y,z (wrapped into [0,L)), molecule, charge, lj_sigma, lj_epsilon,
 *   hal_r0, hal_epsilon, polarizability, hred_parent, hred_factor,
 *   dipole[9*n_mol], quadrupole[18*n_mol].
 * model: 0 = CHARMM-style (config 0), 1 = AMOEBA-style (configs 1-4). */
int mdg_water_generate(int64_t n_mol, double box, uint64_t seed, int model, double* x,
                       double* y, double* z, int32_t* molecule, double* charge,
                       double* lj_sigma, double* lj_epsilon, double* hal_r0,
                       double* hal_epsilon, double* polarizability, int32_t* hred_parent,
                       double* hred_factor, double* dipole, double* quadrupole);
/* Host helper: Halgren-reduced site coordinates, bit-identical to the
 * device's (r_red = r_p + f*wrap1(r_i - r_p), re-wrapped into [0,L)). */
int mdg_reduce_sites_host(int64_t n, double lx, double ly, double lz, const double* x,
                          const double* y, const double* z, const int32_t* parent,
                          const double* factor, double* xr, double* yr, double* zr);

#ifdef __cplusplus
}
#endif
#endif
