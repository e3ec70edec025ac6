// polforce.cu -- polarization forces, torques and pair virial at the
// converged induced dipoles (the epolar1 analogue, no
// counterpart in the reference, whose polarization stops at the solve).
//
// The stationary polarization energy E = 1/2 mu.a^-1.mu - 1/2 mu.T.mu
// - mu.E_perm has the position-dependent pair part (R = r_i - r_j)
//   U_ij = -(h + f + g),  h = mu_i.T_ij.mu_j = rr5 (mu_i.R)(mu_j.R) - rr3 mu_i.mu_j
//   f = mu_i.E_{j->i}(R),  g = mu_j.E_{i->j}(-R)   (skipped for same-molecule
//                                                   pairs: d-scale 0)
// with the Ewald + Thole damped radial functions rr3..rr9 of field_tpre
// (rr_n = B_n - (1 - lambda_n) (2n-1)!!/r^(2n+1)); they obey
// d rr_n / dR = -R rr_(n+2), which gives the closed-form gradients below.
// F_i = -electric dU/dR (mu fixed: Hellmann-Feynman at the solution),
// F_j = -F_i. The permanent multipoles feel the induced dipoles' field:
// torque = (dU/dd) x d plus the quadrupole term of k_mpole. The oracle
// (oracle/mdo.c mdo_polar_forces) differentiates the same energy through
// generic Cartesian tensors and is pinned by finite differences.
#include "common.cuh"

namespace mdg {

struct PFArgs {
  int64_t n_i;
  int ipw;
  const double4* __restrict__ pos;
  const double4* __restrict__ mp;
  const double4* __restrict__ pq4;  // (alpha, alpha^(1/6), q, alpha^(-1/6))
  const double4* __restrict__ mu;
  const int32_t* __restrict__ mol;
  ListView L;
  Box b;
  double c2, alpha, thole_a, electric;
  double4* __restrict__ force;
  double4* __restrict__ torque;
  double* __restrict__ partials;
  int accumulate;
};

struct Sym3 {
  double xx, xy, xz, yy, yz, zz;
};

__device__ __forceinline__ void smul(const Sym3& Q, double x, double y, double z, double& ox,
                                     double& oy, double& oz) {
  ox = Q.xx * x + Q.xy * y + Q.xz * z;
  oy = Q.xy * x + Q.yy * y + Q.yz * z;
  oz = Q.xz * x + Q.yz * y + Q.zz * z;
}

// 2 (M_zy, M_xz, M_yx) with M = Q G - G Q (G = dU/dQ, symmetric): the
// quadrupole torque convention of k_mpole
__device__ __forceinline__ void quad_torque(const Sym3& Q, const Sym3& G, double& tx, double& ty,
                                            double& tz) {
  const double mzy = (Q.xz * G.xy + Q.yz * G.yy + Q.zz * G.yz) - (G.xz * Q.xy + G.yz * Q.yy + G.zz * Q.yz);
  const double mxz = (Q.xx * G.xz + Q.xy * G.yz + Q.xz * G.zz) - (G.xx * Q.xz + G.xy * Q.yz + G.xz * Q.zz);
  const double myx = (Q.xy * G.xx + Q.yy * G.xy + Q.yz * G.xz) - (G.xy * Q.xx + G.yy * Q.xy + G.yz * Q.xz);
  tx += 2.0 * mzy;
  ty += 2.0 * mxz;
  tz += 2.0 * myx;
}

// dU/dQ for U = -e [rr7 s R R^T - rr5 (u R^T + R u^T)] (s = u.R):
__device__ __forceinline__ Sym3 gq(double e, double rr5, double rr7, double s, double ux,
                                   double uy, double uz, double x, double y, double z) {
  const double c = -e * rr7 * s, d = e * rr5;
  return Sym3{c * x * x + d * 2.0 * ux * x,        c * x * y + d * (ux * y + x * uy),
              c * x * z + d * (ux * z + x * uz),    c * y * y + d * 2.0 * uy * y,
              c * y * z + d * (uy * z + y * uz),    c * z * z + d * 2.0 * uz * z};
}

// partial slots: 0 pair energy, 1..9 virial (row-major)
template <bool EXCL, bool PRUNED, bool HALF>
__global__ void __launch_bounds__(kBlock, MDG_POLFORCE_MINB) k_polar_force(PFArgs a) {
  __shared__ double4 ring_mem[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  Ring ring{ring_mem[threadIdx.x >> 5], 0, 0};
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double el = a.electric;
  MDG_SITE_LOOP(i, a.n_i, a.ipw) {
    const double4 pi = a.pos[i];
    const double4 m0i = a.mp[3 * i], m1i = a.mp[3 * i + 1];
    const double qi = a.pq4[i].z;
    const double dix = m0i.x, diy = m0i.y, diz = m0i.z;
    const Sym3 Qi{m0i.w, m1i.x, m1i.y, m1i.z, m1i.w, a.mp[3 * i + 2].x};
    const double4 ui = a.mu[i];
    const double ipdi = a.pq4[i].w;  // 1 / pdamp_i
    const int cnt = a.L.cnt[i];
    const int32_t* row = list_row(a.L, i);
    double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
    auto body = [&](const double4& e) {
      const int32_t raw = ring_j(e);
      const int32_t j = raw & 0x7fffffff;
      const bool excl = EXCL && (raw < 0);  // same molecule (flag set in the prologue)
      const double x = e.x, y = e.y, z = e.z;
      const double r2 = dist2(x, y, z);
      const double4 pj = ldg4(a.pq4 + j);  // (alpha, pdamp, q)
      const double4 uj = ldg4(a.mu + j);
      const double inv_r = rsqrt(r2);  // one MUFU.RSQ64H + Newton, no division
      const double r = r2 * inv_r;
      const double inv_r2 = inv_r * inv_r;
      // Thole lambda3..9 (exponential damping, u = r / (pd_i pd_j))
      const double u = r * ipdi * pj.w;
      const double s1 = a.thole_a * u * u * u;
      const double ex = exp(-s1);
      const double s2 = s1 * s1;
      const double l3 = 1.0 - ex;
      const double l5 = 1.0 - (1.0 + s1) * ex;
      const double l7 = 1.0 - (1.0 + s1 + 0.6 * s2) * ex;
      const double l9 = 1.0 - (1.0 + s1 + (18.0 / 35.0) * s2 + (9.0 / 35.0) * s2 * s1) * ex;
      double bn[5];
      ewald_bn<4>(r, inv_r, inv_r2, a.alpha, bn);
      const double g1 = inv_r2 * inv_r, g2 = 3.0 * g1 * inv_r2, g3 = 5.0 * g2 * inv_r2,
                   g4 = 7.0 * g3 * inv_r2;
      const double rr3 = bn[1] - (1.0 - l3) * g1;
      const double rr5 = bn[2] - (1.0 - l5) * g2;
      const double rr7 = bn[3] - (1.0 - l7) * g3;
      const double rr9 = bn[4] - (1.0 - l9) * g4;

      const double uir = ui.x * x + ui.y * y + ui.z * z;
      const double ujr = uj.x * x + uj.y * y + uj.z * z;
      const double uiuj = ui.x * uj.x + ui.y * uj.y + ui.z * uj.z;
      // h: induced-induced (all pairs)
      double U = rr5 * uir * ujr - rr3 * uiuj;
      const double ch = -rr7 * uir * ujr + rr5 * uiuj;
      double gx = ch * x + rr5 * (ui.x * ujr + uj.x * uir);
      double gy = ch * y + rr5 * (ui.y * ujr + uj.y * uir);
      double gz = ch * z + rr5 * (ui.z * ujr + uj.z * uir);
      double4 m0j = make_double4(0, 0, 0, 0);
      Sym3 Qj{0, 0, 0, 0, 0, 0};
      if (!excl) {
        m0j = ldg4(a.mp + 3 * (size_t)j);
        const double4 m1j = ldg4(a.mp + 3 * (size_t)j + 1);
        Qj = Sym3{m0j.w, m1j.x, m1j.y, m1j.z, m1j.w, __ldg(&a.mp[3 * (size_t)j + 2].x)};
        const double qj = pj.z;
        // f: induced i in the permanent field of j
        double vx, vy, vz, wx, wy, wz;
        smul(Qj, x, y, z, vx, vy, vz);
        smul(Qj, ui.x, ui.y, ui.z, wx, wy, wz);
        const double b = m0j.x * x + m0j.y * y + m0j.z * z;
        const double cq = x * vx + y * vy + z * vz;
        const double md = ui.x * m0j.x + ui.y * m0j.y + ui.z * m0j.z;
        const double mv = ui.x * vx + ui.y * vy + ui.z * vz;
        const double k1 = rr3 * qj + rr5 * b + rr7 * cq;
        U += uir * k1 - rr3 * md - 2.0 * rr5 * mv;
        const double kr = uir * (rr5 * qj + rr7 * b + rr9 * cq) - rr5 * md - 2.0 * rr7 * mv;
        gx += ui.x * k1 + uir * (rr5 * m0j.x + 2.0 * rr7 * vx) - 2.0 * rr5 * wx - kr * x;
        gy += ui.y * k1 + uir * (rr5 * m0j.y + 2.0 * rr7 * vy) - 2.0 * rr5 * wy - kr * y;
        gz += ui.z * k1 + uir * (rr5 * m0j.z + 2.0 * rr7 * vz) - 2.0 * rr5 * wz - kr * z;
        // g: induced j in the permanent field of i (R -> -R)
        double ax, ay, az, cx, cy, cz;
        smul(Qi, x, y, z, ax, ay, az);           // Qi R
        smul(Qi, uj.x, uj.y, uj.z, cx, cy, cz);  // Qi uj
        const double dir = dix * x + diy * y + diz * z;
        const double cqi = x * ax + y * ay + z * az;
        const double mdi = uj.x * dix + uj.y * diy + uj.z * diz;
        const double mvi = uj.x * ax + uj.y * ay + uj.z * az;  // uj.Qi R
        const double k2 = rr3 * qi - rr5 * dir + rr7 * cqi;
        U += -ujr * k2 - rr3 * mdi + 2.0 * rr5 * mvi;
        const double kr2 = -ujr * (rr5 * qi - rr7 * dir + rr9 * cqi) - rr5 * mdi + 2.0 * rr7 * mvi;
        gx += -uj.x * k2 + ujr * (rr5 * dix - 2.0 * rr7 * ax) + 2.0 * rr5 * cx - kr2 * x;
        gy += -uj.y * k2 + ujr * (rr5 * diy - 2.0 * rr7 * ay) + 2.0 * rr5 * cy - kr2 * y;
        gz += -uj.z * k2 + ujr * (rr5 * diz - 2.0 * rr7 * az) + 2.0 * rr5 * cz - kr2 * z;
        // torque on i's permanent multipoles (from g): dU/dd_i, dU/dQ_i
        {
          const double hx = -el * (rr5 * ujr * x - rr3 * uj.x);
          const double hy = -el * (rr5 * ujr * y - rr3 * uj.y);
          const double hz = -el * (rr5 * ujr * z - rr3 * uj.z);
          tx += hy * diz - hz * diy;
          ty += hz * dix - hx * diz;
          tz += hx * diy - hy * dix;
          quad_torque(Qi, gq(el, rr5, rr7, -ujr, -uj.x, -uj.y, -uj.z, x, y, z), tx, ty, tz);
        }
      }
      const bool jside = HALF && j < a.n_i;
      const double w = (HALF && !jside) ? 0.5 : 1.0;
      acc[0] += w * (-el * U);
      // F_i = electric * grad(h + f + g)
      const double Fx = el * gx, Fy = el * gy, Fz = el * gz;
      fx += Fx;
      fy += Fy;
      fz += Fz;
      acc[1] += w * (x * Fx);
      acc[2] += w * (x * Fy);
      acc[3] += w * (x * Fz);
      acc[4] += w * (y * Fx);
      acc[5] += w * (y * Fy);
      acc[6] += w * (y * Fz);
      acc[7] += w * (z * Fx);
      acc[8] += w * (z * Fy);
      acc[9] += w * (z * Fz);
      if (jside) {
        atomicAdd(&a.force[j].x, -Fx);
        atomicAdd(&a.force[j].y, -Fy);
        atomicAdd(&a.force[j].z, -Fz);
        if (!excl) {  // torque on j's permanent multipoles (from f)
          const double hx = -el * (rr5 * uir * x - rr3 * ui.x);
          const double hy = -el * (rr5 * uir * y - rr3 * ui.y);
          const double hz = -el * (rr5 * uir * z - rr3 * ui.z);
          double ux = hy * m0j.z - hz * m0j.y;
          double uy = hz * m0j.x - hx * m0j.z;
          double uz = hx * m0j.y - hy * m0j.x;
          quad_torque(Qj, gq(el, rr5, rr7, uir, ui.x, ui.y, ui.z, x, y, z), ux, uy, uz);
          atomicAdd(&a.torque[j].x, ux);
          atomicAdd(&a.torque[j].y, uy);
          atomicAdd(&a.torque[j].z, uz);
        }
      }
    };
    const int start = (HALF && a.L.sorted) ? row_suffix(row, cnt, i, lane) : 0;
    run_row<false, PRUNED>(
        row + start, cnt - start, lane, a.pos, nullptr, ring,
        [&](int32_t& raw, const double4& pj, int32_t, double& x, double& y, double& z) {
          const int32_t j = raw & 0x7fffffff;
          const double r2 = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, x, y, z);
          bool keep;
          if (PRUNED) {
            keep = true;  // pruned rows: in range, flag already set
          } else {
            keep = r2 <= a.c2;
            raw = (EXCL && same_group(pj, pi)) ? (j | (int32_t)0x80000000) : j;  // w: group
          }
          return keep && !(HALF && j < i);
        },
        [&](const double4& e, int) { body(e); });
    fx = warp_allsum(fx);
    fy = warp_allsum(fy);
    fz = warp_allsum(fz);
    tx = warp_allsum(tx);
    ty = warp_allsum(ty);
    tz = warp_allsum(tz);
    if (lane == 0) {
      if (HALF) {  // force / torque hold their accumulated base (or zero)
        atomicAdd(&a.force[i].x, fx);
        atomicAdd(&a.force[i].y, fy);
        atomicAdd(&a.force[i].z, fz);
        atomicAdd(&a.torque[i].x, tx);
        atomicAdd(&a.torque[i].y, ty);
        atomicAdd(&a.torque[i].z, tz);
      } else {
        if (a.accumulate) {
          const double4 f0 = a.force[i], t0 = a.torque[i];
          fx += f0.x;
          fy += f0.y;
          fz += f0.z;
          tx += t0.x;
          ty += t0.y;
          tz += t0.z;
        }
        a.force[i] = make_double4(fx, fy, fz, 0.0);
        a.torque[i] = make_double4(tx, ty, tz, 0.0);
      }
    }
  }
  block_store_partials<10>(acc, a.partials);
}

template <bool PRUNED>
static void launch_polar_force(mdg_ctx* c, PFArgs& k, bool ex, bool half) {
  constexpr int slot = 70;
  if (!half) {
    if (ex) MDG_LAUNCH_SITES(c, "polar_force", k.n_i, k, (k_polar_force<true, PRUNED, false>));
    else MDG_LAUNCH_SITES(c, "polar_force", k.n_i, k, (k_polar_force<false, PRUNED, false>));
    finalize_partials(c, c->last_grid, 10, slot, 0.5);
    return;
  }
  const size_t bytes = (size_t)k.n_i * sizeof(double4);
  if (!k.accumulate) {
    MDG_CUDA_CHECK(cudaMemsetAsync(k.force, 0, bytes, c->stream));
    MDG_CUDA_CHECK(cudaMemsetAsync(k.torque, 0, bytes, c->stream));
  }
  if (ex) MDG_LAUNCH_SITES(c, "polar_force", k.n_i, k, (k_polar_force<true, PRUNED, true>));
  else MDG_LAUNCH_SITES(c, "polar_force", k.n_i, k, (k_polar_force<false, PRUNED, true>));
  finalize_partials(c, c->last_grid, 10, slot, 1.0);
}

static PFArgs pf_args(mdg_ctx* c, double alpha, double thole_a, double electric, bool accumulate) {
  PFArgs k;
  k.n_i = c->n_own;
  k.pos = c->pos;
  k.mp = c->mp;
  k.pq4 = c->pq4;
  k.mu = c->mu;
  k.mol = c->mol;
  k.b = make_box(c->lx, c->ly, c->lz);
  k.alpha = alpha;
  k.thole_a = thole_a;
  k.electric = electric;
  k.force = c->force;
  k.torque = c->torque;
  k.accumulate = accumulate ? 1 : 0;
  return k;
}

void run_polar_force(mdg_ctx* c, int list_id, double alpha, double cutoff, double thole_a,
                     double electric, int exclude, bool accumulate) {
  const DevList& L = c->lists[list_id];
  PFArgs k = pf_args(c, alpha, thole_a, electric, accumulate);
  k.L = kernel_rows(c, list_id, cutoff);
  k.c2 = cutoff * cutoff;
  launch_polar_force<false>(c, k, exclude && c->has_mol, !c->deterministic);
}

void run_polar_force_pruned(mdg_ctx* c, double alpha, double thole_a, double electric,
                            int exclude, bool accumulate) {
  const PrunedList& P = c->plist;
  PFArgs k = pf_args(c, alpha, thole_a, electric, accumulate);
  k.L = ListView{P.nbr, P.cnt, P.cap, P.sorted};
  k.c2 = P.cutoff * P.cutoff;
  // the pruned rows carry the same-molecule flag only when written with
  // exclusions (field_tpre with exclude): EXCL follows the request
  launch_polar_force<true>(c, k, exclude && c->has_mol, !c->deterministic);
}

}  // namespace mdg
