/*
 * mdo.h -- CPU ORACLE (test infrastructure only; never linked into the product).
 *
 * Plain-C restatement of the reference `mdvec` real-space pair path
 * (/root/reference/proj, read-only) plus the north-star extensions the
 * reference lacks (exclusions, virial, electric constant, Halgren H-reduction,
 * Ewald-damped Thole field and T, real-space multipole Ewald, PCG).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the CPU baseline. Each function cites the reference file:line it follows;
 * functions marked "EXTENSION" have no reference counterpart and are pinned
 * by the limit tests named in DESIGN.md (alpha -> 0, multipoles -> charges,
 * finite differences, dense solves).
 *
 * Conventions (same as the reference):
 *  - arrays are in the caller's (original) site order, SoA, double;
 *  - displacement d = r_i - r_j wrapped by wrap1 into [-L/2, L/2);
 *  - force scalar fs: F_i = fs * d (reference proj/include/mdvec/kernels.hpp:37-40);
 *  - outputs are OVERWRITTEN (reference `out.reset()`, kernels_scalar.cpp:13);
 *  - status codes: 0 OK, 1 CONTRACT, 2 CAPACITY, 3 SINGULARITY, 4 CONVERGENCE.
 */
#ifndef MDO_H
#define MDO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MDO_OK = 0, MDO_CONTRACT = 1, MDO_CAPACITY = 2, MDO_SINGULARITY = 3,
       MDO_CONVERGENCE = 4 };

#define MDO_MAX_NEIGHBORS 2560 /* proj/include/mdvec/common.hpp:10 */

/* Site data (reference ParticleSystem, proj/include/mdvec/system.hpp:12-25)
 * plus the extension arrays. Any extension pointer may be NULL. */
typedef struct {
  size_t n;
  double lx, ly, lz;
  const double *x, *y, *z;
  const double *charge, *lj_sigma, *lj_epsilon, *hal_r0, *hal_epsilon, *polarizability;
  const int32_t *molecule; /* EXTENSION: exclusion groups (NULL = no exclusions) */
  const double *dipole;    /* EXTENSION: 3n, (mux,muy,muz) per site */
  const double *quadrupole;/* EXTENSION: 6n traceless (xx,xy,xz,yy,yz,zz) per site */
} mdo_system;

/* Reference NeighborTable (proj/include/mdvec/neighbors.hpp:25-41). */
typedef struct {
  size_t n_sites;
  double cutoff;
  uint32_t *nnvlst, *nvloop8, *nvloop16;
  uint64_t *offset;
  int32_t *indices;
  double *scale;
  size_t total; /* total padded slots */
} mdo_table;

const char* mdo_last_error(void);

/* ---- geometry: proj/include/mdvec/pbc.hpp:27-37 ------------------------ */
double mdo_wrap1(double d, double box_len, double inv_len, double half_len);
double mdo_dist2(double dx, double dy, double dz);
int mdo_minimum_image(double* dx, double* dy, double* dz, double lx, double ly, double lz);

/* ---- reference generator restatement: proj/src/system.cpp:65-190 ------- */
/* kind 0 = lattice-water-like, 1 = uniform-random. Out arrays length n. */
int mdo_generate_system(int kind, size_t n, double lx, double ly, double lz, uint64_t seed,
                        double min_separation, double* x, double* y, double* z, double* charge,
                        double* lj_sigma, double* lj_epsilon, double* hal_r0,
                        double* hal_epsilon, double* polarizability);
void mdo_random_dipoles(size_t n, uint64_t seed, double magnitude, double* mx, double* my,
                        double* mz);

/* ---- neighbour lists: proj/src/neighbors.cpp, neighbors_vec.cpp -------- */
int mdo_table_build(const mdo_system* s, double list_cutoff, size_t extra_pad, mdo_table* out);
void mdo_table_free(mdo_table* t);
/* Canonical sorted (i<j) pairs, brute force O(N^2) (neighbors.cpp:38-57). out
 * must hold 2*cap int32; *npairs receives the count (CAPACITY if > cap). */
int mdo_brute_force_pairs(const mdo_system* s, double cutoff, int32_t* out, size_t cap,
                          size_t* npairs);
/* Full rows of the listed sites, brute force with the reference predicate. */
int mdo_rows_for_sites(const mdo_system* s, double cutoff, const int32_t* sites, size_t ns,
                       int32_t* counts, int32_t* idx, size_t cap);
int mdo_table_pairs(const mdo_table* t, int32_t* out, size_t cap, size_t* npairs);

/* ---- nonpolar kernels (kernels_scalar.cpp:10-94, polar_scalar.cpp:26-67) */
/* exclude != 0 skips pairs with equal molecule ids (EXTENSION).
 * electric scales the Coulomb energy/force (EXTENSION; 1.0 = reference).
 * virial (9, row-major, may be NULL) = sum over pairs of d (x) F_i (EXTENSION). */
int mdo_lj(const mdo_system* s, const mdo_table* t, double cutoff, int shift, int exclude,
           double* fx, double* fy, double* fz, double* energy, double* virial);
int mdo_ewald_real(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                   double electric, int exclude, double* fx, double* fy, double* fz,
                   double* energy, double* virial);
int mdo_halgren(const mdo_system* s, const mdo_table* t, double cutoff, double delta,
                double gamma, int exclude, double* fx, double* fy, double* fz,
                double* energy, double* virial);

/* ---- reference polar kernels (polar_scalar.cpp:69-198) ----------------- */
int mdo_tmatvec_thole(const mdo_system* s, const mdo_table* t, double cutoff, double thole_a,
                      const double* mx, const double* my, const double* mz, double* ex,
                      double* ey, double* ez);
int mdo_perm_field_thole(const mdo_system* s, const mdo_table* t, double cutoff,
                         double thole_a, double* ex, double* ey, double* ez);
int mdo_jacobi(const mdo_system* s, const mdo_table* t, double cutoff, double thole_a,
               double tol, size_t max_iter, double* mx, double* my, double* mz,
               double* last_residual, size_t* iters);

/* ---- EXTENSIONS (no reference counterpart) ----------------------------- */
/* Halgren H-reduction sites: r_red = r_p + f * wrap1(r_i - r_p), re-wrapped
 * into [0, L) (Tinker-HP convention; SURVEY 8(c) gap ledger). */
/* BASELINE.json 3-site water fixture (same contract as mdg_water_generate). */
int mdo_water_generate(int64_t n_mol, double box, uint64_t seed, int model, double* x,
                       double* y, double* z, int32_t* molecule, double* charge,
                       double* lj_sigma, double* lj_epsilon, double* hal_r0,
                       double* hal_epsilon, double* polarizability, int32_t* hred_parent,
                       double* hred_factor, double* dipole, double* quadrupole);
void mdo_reduce_sites(size_t n, const double* x, const double* y, const double* z,
                      const int32_t* parent, const double* factor, double lx, double ly,
                      double lz, double* xr, double* yr, double* zr);
/* Chain rule: F_i += f_i * Fred_i, F_parent += (1 - f_i) * Fred_i. Overwrites f*. */
void mdo_reduce_forces(size_t n, const int32_t* parent, const double* factor,
                       const double* frx, const double* fry, const double* frz, double* fx,
                       double* fy, double* fz);

/* Ewald radial functions B_0..B_nmax (Tinker bn recursion). */
void mdo_ewald_bn(double r, double alpha, int nmax, double* bn);

/* Real-space Ewald + Thole T mat-vec, all list pairs within cutoff (u-scale 1).
 * Reduces exactly to mdo_tmatvec_thole at alpha = 0. */
int mdo_tmatvec_ewald(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                      double thole_a, const double* mu /*3n*/, double* e /*3n*/);
/* Permanent field of q + mu + Theta, real-space Ewald + Thole (lambda3/5/7),
 * pairs of one molecule excluded when exclude != 0 (d-scale 0). Reduces to
 * mdo_perm_field_thole at alpha = 0 with dipoles/quadrupoles zero. */
int mdo_perm_field_ewald(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                         double thole_a, int exclude, double* e /*3n*/);
/* Real-space multipole Ewald energy, forces, torques and pair virial, from
 * the generic Cartesian interaction tensors T^(0..5) of B_n(r). */
int mdo_mpole(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
              double electric, int exclude, double* f /*3n*/, double* torque /*3n*/,
              double* energy, double* virial);
/* Field from the tensor form, no Thole (checks mdo_perm_field_ewald's
 * thole->off limit). */
int mdo_mpole_field_tensor(const mdo_system* s, const mdo_table* t, double alpha,
                           double cutoff, int exclude, double* e /*3n*/);

/* Polarization forces at fixed induced dipoles mu (EXTENSION, SURVEY 8(f)#1,
 * the epolar1 analogue). With the variational energy
 *   E(mu) = 1/2 mu.alpha^-1.mu - 1/2 mu.T.mu - mu.E_perm
 * (stationary at the PCG solution, where E = -1/2 mu.E_perm), the force is
 * -dE/dr at fixed mu: pair energy U_ij = -mu_i.T_ij.mu_j - mu_i.E_{j->i}
 * - mu_j.E_{i->j} with the Ewald + Thole damped radial functions of T and
 * the permanent field (the field terms skipped for same-molecule pairs when
 * exclude != 0), differentiated through the generic Cartesian tensors.
 * energy = electric * sum U_ij (the mu-dependent part, add
 * 1/2 mu.alpha^-1.mu for E); torque = torques on the permanent multipoles
 * from the induced dipoles' field. */
int mdo_polar_forces(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                     double thole_a, double electric, int exclude, const double* mu /*3n*/,
                     double* f /*3n*/, double* torque /*3n*/, double* energy, double* virial);

/* Diagonal-preconditioned CG for (alpha^-1 - T) mu = E_perm with
 * mdo_tmatvec_ewald as T. mu0 = alpha E. Converged when
 * sqrt(sum |dmu|^2 / n) * debye < tol_debye. */
int mdo_pcg(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
            double thole_a, const double* eperm /*3n*/, double tol_debye, size_t max_iter,
            double* mu /*3n*/, size_t* iters, double* last_rms_debye);

#define MDO_DEBYE 4.80321
#define MDO_ELECTRIC 332.063713

#ifdef __cplusplus
}
#endif
#endif
