// md.cu -- the MD time loop around the force kernels:
// harmonic bonded terms for flexible molecules and the device-resident
// integrator steps -- kick (B), drift (A) and the Langevin velocity update
// (O) -- that mdg_md_run composes into velocity Verlet or a two-level
// BAOAB-RESPA (the multi-timestep scheme of /root/reference/PAPER.md:782-783,
// bonded terms in the inner level), so a trajectory runs without host round
// trips for coordinates.
//
// Units: kcal/mol, A, amu, fs. a = F/m * kAccel with kAccel = 4.184e-4
// (1 kcal/mol = 4.184e-4 amu A^2 / fs^2). Bond energy k (r - r0)^2, angle
// energy k (theta - theta0)^2 (Tinker's harmonic convention, no 1/2).
#include "common.cuh"

namespace mdg {

constexpr double kAccel = 4.184e-4;

__device__ __forceinline__ void add_force(double4* f, int i, double x, double y, double z) {
  atomicAdd(&f[i].x, x);
  atomicAdd(&f[i].y, y);
  atomicAdd(&f[i].z, z);
}

// partial slot 0: bond energy
__global__ void __launch_bounds__(kBlock) k_bonds(int64_t nb, Box b, const double4* __restrict__ pos,
                                                 const int2* __restrict__ ij,
                                                 const double2* __restrict__ par,
                                                 double4* __restrict__ force,
                                                 double* __restrict__ partials) {
  double acc[1] = {0.0};
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nb) {
    const int2 e = ij[k];
    const double2 p = par[k];
    const double4 pi = pos[e.x], pj = pos[e.y];
    double dx, dy, dz;
    const double r = sqrt(min_image(b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, dx, dy, dz));
    const double dr = r - p.y;
    acc[0] = p.x * dr * dr;
    const double s = -2.0 * p.x * dr / r;  // F_i = -dE/dr_i
    add_force(force, e.x, s * dx, s * dy, s * dz);
    add_force(force, e.y, -s * dx, -s * dy, -s * dz);
  }
  block_store_partials<1>(acc, partials);
}

// angle (i, j vertex, k); partial slot 0: angle energy
__global__ void __launch_bounds__(kBlock) k_angles(int64_t na, Box b, const double4* __restrict__ pos,
                                                  const int4* __restrict__ ijk,
                                                  const double2* __restrict__ par,
                                                  double4* __restrict__ force,
                                                  double* __restrict__ partials) {
  double acc[1] = {0.0};
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < na) {
    const int4 e = ijk[t];
    const double2 p = par[t];
    const double4 pi = pos[e.x], pj = pos[e.y], pk = pos[e.z];
    double ax, ay, az, cx, cy, cz;
    min_image(b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, ax, ay, az);  // a = r_i - r_j
    min_image(b, pk.x, pk.y, pk.z, pj.x, pj.y, pj.z, cx, cy, cz);  // c = r_k - r_j
    const double ra2 = ax * ax + ay * ay + az * az, rc2 = cx * cx + cy * cy + cz * cz;
    const double ra = sqrt(ra2), rc = sqrt(rc2);
    double cs = (ax * cx + ay * cy + az * cz) / (ra * rc);
    cs = fmin(1.0, fmax(-1.0, cs));
    const double th = acos(cs);
    const double dth = th - p.y;
    acc[0] = p.x * dth * dth;
    // dE/dtheta, dtheta/da = -(c/(ra rc) - cs a/ra^2) / sin
    const double sn = fmax(sqrt(fmax(0.0, 1.0 - cs * cs)), 1e-12);
    const double de = 2.0 * p.x * dth;
    const double fa = de / (sn * ra);  // F_i = -dE/dtheta * dtheta/dr_i
    const double fc = de / (sn * rc);
    const double fix = fa * (cx / rc - cs * ax / ra), fiy = fa * (cy / rc - cs * ay / ra),
                 fiz = fa * (cz / rc - cs * az / ra);
    const double fkx = fc * (ax / ra - cs * cx / rc), fky = fc * (ay / ra - cs * cy / rc),
                 fkz = fc * (az / ra - cs * cz / rc);
    add_force(force, e.x, fix, fiy, fiz);
    add_force(force, e.z, fkx, fky, fkz);
    add_force(force, e.y, -fix - fkx, -fiy - fky, -fiz - fkz);
  }
  block_store_partials<1>(acc, partials);
}

// v += F / m * dt/2 ; vel.w = 1/m (amu^-1)
__global__ void k_kick(int64_t n, double hdt, const double4* __restrict__ force,
                       double4* __restrict__ vel) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 v = vel[i];
  const double4 f = force[i];
  const double s = hdt * kAccel * v.w;
  v.x += s * f.x;
  v.y += s * f.y;
  v.z += s * f.z;
  vel[i] = v;
}

// Counter-based normal deviates for the Langevin O step, reproducible on the
// host (oracle/md.py restates them): SplitMix64 of (seed, step counter,
// caller site id, component) -> two 32-bit uniforms -> Box-Muller.
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double gauss(uint64_t key) {
  const uint64_t h = splitmix64(key);
  const double u1 = (double)((h >> 32) + 1) * 0x1p-32;  // (0, 1]
  const double u2 = (double)(h & 0xffffffffull) * 0x1p-32;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

// O: v = c1 v + c2 sqrt(kT/m) xi (kt_acc = kB T * kAccel; vel.w = 1/m)
__global__ void k_ostep(int64_t n, double c1, double c2, double kt_acc, uint64_t seed,
                        uint64_t counter, const int32_t* __restrict__ perm,
                        double4* __restrict__ vel) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 v = vel[i];
  const double s = c2 * sqrt(kt_acc * v.w);
  const uint64_t base = splitmix64(seed + splitmix64(counter)) + 3ull * (uint64_t)perm[i];
  v.x = c1 * v.x + s * gauss(base);
  v.y = c1 * v.y + s * gauss(base + 1);
  v.z = c1 * v.z + s * gauss(base + 2);
  vel[i] = v;
}

__device__ __forceinline__ double wrap_box(double p, double L) {
  p -= L * floor(p / L);
  return (p >= L || p < 0.0) ? 0.0 : p;
}

// x += v dt, wrapped into [0, L) (the engine's position contract)
__global__ void k_drift(int64_t n, double dt, Box b, const double4* __restrict__ vel,
                        double4* __restrict__ pos, double4* __restrict__ vsite, int copy_vsite) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 v = vel[i];
  double4 p = pos[i];
  p.x = wrap_box(p.x + dt * v.x, b.lx);
  p.y = wrap_box(p.y + dt * v.y, b.ly);
  p.z = wrap_box(p.z + dt * v.z, b.lz);
  pos[i] = p;
  if (copy_vsite) vsite[i] = p;
}

// kinetic energy (kcal/mol): 1/2 m v^2 / kAccel
__global__ void __launch_bounds__(kBlock) k_kinetic(int64_t n, const double4* __restrict__ vel,
                                                   double* __restrict__ partials) {
  double acc[1] = {0.0};
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double4 v = vel[i];
    if (v.w > 0) acc[0] = 0.5 * (v.x * v.x + v.y * v.y + v.z * v.z) / (v.w * kAccel);
  }
  block_store_partials<1>(acc, partials);
}

// results: 100 bond energy, 101 angle energy, 102 kinetic energy
void run_bonded(mdg_ctx* c) { run_bonded(c, c->force); }

void run_bonded(mdg_ctx* c, double4* out) {
  const Box b = make_box(c->lx, c->ly, c->lz);
  ensure_partials(c, std::max(grid_for(c->nbonds), grid_for(c->nangles)));
  if (c->nbonds > 0) {
    MDG_LAUNCH(c, "bonds", grid_for(c->nbonds), kBlock, 0, k_bonds, c->nbonds, b, c->pos,
               c->bond_ij, c->bond_par, out, c->partials);
    finalize_partials(c, grid_for(c->nbonds), 1, 100, 1.0);
  }
  if (c->nangles > 0) {
    MDG_LAUNCH(c, "angles", grid_for(c->nangles), kBlock, 0, k_angles, c->nangles, b, c->pos,
               c->angle_ijk, c->angle_par, out, c->partials);
    finalize_partials(c, grid_for(c->nangles), 1, 101, 1.0);
  }
}

void run_kick(mdg_ctx* c, double half_dt) { run_kick(c, half_dt, c->force); }

void run_kick(mdg_ctx* c, double half_dt, const double4* force) {
  MDG_LAUNCH(c, "kick", grid_for(c->n, 256), 256, 0, k_kick, c->n, half_dt, force, c->vel);
}

void run_ostep(mdg_ctx* c, double c1, double kt, uint64_t seed, uint64_t counter) {
  MDG_LAUNCH(c, "ostep", grid_for(c->n, 256), 256, 0, k_ostep, c->n, c1,
             std::sqrt(std::max(0.0, 1.0 - c1 * c1)), kt * kAccel, seed, counter, c->d_perm,
             c->vel);
}

void run_drift(mdg_ctx* c, double dt) {
  MDG_LAUNCH(c, "drift", grid_for(c->n, 256), 256, 0, k_drift, c->n, dt,
             make_box(c->lx, c->ly, c->lz), c->vel, c->pos, c->vsite, c->has_hred ? 0 : 1);
  if (c->has_hred) run_reduce_sites(c);
}

void run_kinetic(mdg_ctx* c) {
  ensure_partials(c, grid_for(c->n));
  MDG_LAUNCH(c, "kinetic", grid_for(c->n), kBlock, 0, k_kinetic, c->n, c->vel, c->partials);
  finalize_partials(c, grid_for(c->n), 1, 102, 1.0);
}

}  // namespace mdg
