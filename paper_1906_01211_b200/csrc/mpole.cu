// mpole.cu -- real-space Ewald permanent-multipole energy, forces, torques
// and pair virial (the empole1 analogue; no counterpart in the reference,
// which covers charges only: SPEC.md:9).
//
// Pair energy with R = r_i - r_j and G_n = B_n(R) (Ewald bn recursion):
//   U = C0 G0 + C1 G1 + C2 G2 + C3 G3 + C4 G4
//   C0 = qi qj
//   C1 = qi dj.R - qj di.R + di.dj
//   C2 = qi R.Qj.R + qj R.Qi.R - (di.R)(dj.R) + 2 (di.QjR - dj.QiR + Qi:Qj)
//   C3 = -(di.R)(R.Qj.R) + (R.Qi.R)(dj.R) - 4 (QiR).(QjR)
//   C4 = (R.Qi.R)(R.Qj.R)
// (Tinker's stored quadrupole Q = Theta/3.) dG_n/dR = -R G_{n+1} gives the
// force F_i = -dU/dR; the torque on i is -mu_i x dU/dmu_i plus the
// quadrupole term from dU/dQ_i. The oracle (oracle/mdo.c mdo_mpole) computes
// the same quantities from generic Cartesian T-tensors instead.
#include "common.cuh"

namespace mdg {

struct MKArgs {
  int64_t n_i;
  int ipw;
  const double4* __restrict__ pos;
  const double4* __restrict__ mp;
  const double4* __restrict__ pq4;  // charges (z)
  const int32_t* __restrict__ mol;
  ListView L;
  Box b;
  double c2, alpha, electric;
  double4* __restrict__ force;
  double4* __restrict__ torque;
  double* __restrict__ partials;
  int accumulate;  // force/torque += instead of =
};

struct Quad {
  double xx, xy, xz, yy, yz, zz;
};

__device__ __forceinline__ void qmul(const Quad& Q, double x, double y, double z, double& ox,
                                     double& oy, double& oz) {
  ox = Q.xx * x + Q.xy * y + Q.xz * z;
  oy = Q.xy * x + Q.yy * y + Q.yz * z;
  oz = Q.xz * x + Q.yz * y + Q.zz * z;
}

// partial slots: 0 energy, 1..9 virial (row-major)
// HALF (default): each owned-owned pair once, in the row of its lower sorted
// index; the partner gets F_j = -F_i and its own torque (the i-side formulas
// with i <-> j and R -> -R) through FP64 atomics. Halo pairs stay in the
// owned row at energy/virial weight 1/2. !HALF: full rows, no atomics.
template <bool EXCL, bool PRUNED, bool HALF>
__global__ void __launch_bounds__(kBlock, MDG_MPOLE_MINB) k_mpole(MKArgs a) {
  __shared__ double4 ring_mem[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  Ring ring{ring_mem[threadIdx.x >> 5], 0, 0};
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  MDG_SITE_LOOP(i, a.n_i, a.ipw) {
    const double4 pi = a.pos[i];
    // i's multipole times the electric constant: every output is linear in
    // it, so the pair factors G_n need no scaling (6 multiplies per pair)
    const double ec = a.electric;
    const double4 m0i = a.mp[3 * i], m1i = a.mp[3 * i + 1];
    const double qi = ec * a.pq4[i].z;
    const double dix = ec * m0i.x, diy = ec * m0i.y, diz = ec * m0i.z;
    const Quad Qi{ec * m0i.w, ec * m1i.x, ec * m1i.y, ec * m1i.z, ec * m1i.w,
                  ec * a.mp[3 * i + 2].x};
    const int cnt = a.L.cnt[i];
    const int32_t* row = list_row(a.L, i);
    double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
    auto body = [&](const double4& e) {
      const int32_t j = ring_j(e);
      const double x = e.x, y = e.y, z = e.z;
      const double r2 = dist2(x, y, z);
      const double qj = __ldg(&a.pq4[j].z);
      const double4 m0j = ldg4(a.mp + 3 * (size_t)j), m1j = ldg4(a.mp + 3 * (size_t)j + 1);
      const Quad Qj{m0j.w, m1j.x, m1j.y, m1j.z, m1j.w, __ldg(&a.mp[3 * (size_t)j + 2].x)};
      const double djx = m0j.x, djy = m0j.y, djz = m0j.z;
      const double inv_r = rsqrt(r2);  // one MUFU.RSQ64H + Newton, no division
      const double r = r2 * inv_r;
      const double inv_r2 = inv_r * inv_r;
      double G[6];
      ewald_bn<5>(r, inv_r, inv_r2, a.alpha, G);

      double vix, viy, viz, vjx, vjy, vjz;
      qmul(Qi, x, y, z, vix, viy, viz);
      qmul(Qj, x, y, z, vjx, vjy, vjz);
      const double dir = dix * x + diy * y + diz * z;
      const double djr = djx * x + djy * y + djz * z;
      const double qir = x * vix + y * viy + z * viz;
      const double qjr = x * vjx + y * vjy + z * vjz;
      const double dij = dix * djx + diy * djy + diz * djz;
      const double diqj = dix * vjx + diy * vjy + diz * vjz;
      const double djqi = djx * vix + djy * viy + djz * viz;
      const double qiqj = Qi.xx * Qj.xx + Qi.yy * Qj.yy + Qi.zz * Qj.zz +
                          2.0 * (Qi.xy * Qj.xy + Qi.xz * Qj.xz + Qi.yz * Qj.yz);
      const double qvv = vix * vjx + viy * vjy + viz * vjz;
      const double C0 = qi * qj;
      const double C1 = qi * djr - qj * dir + dij;
      const double C2 = qi * qjr + qj * qir - dir * djr + 2.0 * (diqj - djqi + qiqj);
      const double C3 = -dir * qjr + qir * djr - 4.0 * qvv;
      const double C4 = qir * qjr;
      const bool jside = HALF && j < a.n_i;
      const double w = (HALF && !jside) ? 0.5 : 1.0;
      acc[0] += w * (C0 * G[0] + C1 * G[1] + C2 * G[2] + C3 * G[3] + C4 * G[4]);

      // gradient dU/dR
      double a1x, a1y, a1z, a2x, a2y, a2z, b1x, b1y, b1z, b2x, b2y, b2z;
      qmul(Qj, dix, diy, diz, a1x, a1y, a1z);  // Qj di
      qmul(Qi, djx, djy, djz, a2x, a2y, a2z);  // Qi dj
      qmul(Qi, vjx, vjy, vjz, b1x, b1y, b1z);  // Qi vj
      qmul(Qj, vix, viy, viz, b2x, b2y, b2z);  // Qj vi
      const double s = C0 * G[1] + C1 * G[2] + C2 * G[3] + C3 * G[4] + C4 * G[5];
      const double gx = G[1] * (qi * djx - qj * dix) +
                        G[2] * (2.0 * (qi * vjx + qj * vix) - djr * dix - dir * djx +
                                2.0 * (a1x - a2x)) +
                        G[3] * (-qjr * dix - 2.0 * dir * vjx + 2.0 * djr * vix + qir * djx -
                                4.0 * (b1x + b2x)) +
                        G[4] * 2.0 * (qjr * vix + qir * vjx) - s * x;
      const double gy = G[1] * (qi * djy - qj * diy) +
                        G[2] * (2.0 * (qi * vjy + qj * viy) - djr * diy - dir * djy +
                                2.0 * (a1y - a2y)) +
                        G[3] * (-qjr * diy - 2.0 * dir * vjy + 2.0 * djr * viy + qir * djy -
                                4.0 * (b1y + b2y)) +
                        G[4] * 2.0 * (qjr * viy + qir * vjy) - s * y;
      const double gz = G[1] * (qi * djz - qj * diz) +
                        G[2] * (2.0 * (qi * vjz + qj * viz) - djr * diz - dir * djz +
                                2.0 * (a1z - a2z)) +
                        G[3] * (-qjr * diz - 2.0 * dir * vjz + 2.0 * djr * viz + qir * djz -
                                4.0 * (b1z + b2z)) +
                        G[4] * 2.0 * (qjr * viz + qir * vjz) - s * z;
      fx -= gx;
      fy -= gy;
      fz -= gz;
      acc[1] -= w * (x * gx);
      acc[2] -= w * (x * gy);
      acc[3] -= w * (x * gz);
      acc[4] -= w * (y * gx);
      acc[5] -= w * (y * gy);
      acc[6] -= w * (y * gz);
      acc[7] -= w * (z * gx);
      acc[8] -= w * (z * gy);
      acc[9] -= w * (z * gz);

      // dipole torque: tau = gmu x di, gmu = dU/d(di)
      const double c1 = G[1] * qj + G[2] * djr + G[3] * qjr;  // coefficient of -R
      const double gmx = G[1] * djx + 2.0 * G[2] * vjx - c1 * x;
      const double gmy = G[1] * djy + 2.0 * G[2] * vjy - c1 * y;
      const double gmz = G[1] * djz + 2.0 * G[2] * vjz - c1 * z;
      tx += gmy * diz - gmz * diy;
      ty += gmz * dix - gmx * diz;
      tz += gmx * diy - gmy * dix;
      // quadrupole torque: GQ = dU/dQi (symmetric), tau = 2 axial(Qi GQ - GQ Qi)
      // with axial(M) = (M_zy, M_xz, M_yx). GQ = crr RR' - G2 (dj R' + R dj')
      // + 2 G2 Qj - 2 G3 (R vj' + vj R'), and for a symmetric u v' + v u' the
      // axial vector is v x (Qi u) + u x (Qi v), so
      //   tau/2 = crr R x vi - G2 (R x Qi dj + dj x vi) + 2 G2 X
      //           - 2 G3 (vj x vi + R x Qi vj),  X = axial(Qi Qj - Qj Qi).
      // (The partner: the same with i <-> j, R -> -R; X changes sign.)
      const double crr = G[2] * qj + G[3] * djr + G[4] * qjr;  // coefficient of R R^T
      const double Xx = (Qi.xz * Qj.xy + Qi.yz * Qj.yy + Qi.zz * Qj.yz) -
                        (Qj.xz * Qi.xy + Qj.yz * Qi.yy + Qj.zz * Qi.yz);
      const double Xy = (Qi.xx * Qj.xz + Qi.xy * Qj.yz + Qi.xz * Qj.zz) -
                        (Qj.xx * Qi.xz + Qj.xy * Qi.yz + Qj.xz * Qi.zz);
      const double Xz = (Qi.xy * Qj.xx + Qi.yy * Qj.xy + Qi.yz * Qj.xz) -
                        (Qj.xy * Qi.xx + Qj.yy * Qi.xy + Qj.yz * Qi.xz);
      const double g2 = 2.0 * G[2], g3 = 2.0 * G[3];
      // vj x vi (the partner uses vi x vj = -(vj x vi))
      const double wx = vjy * viz - vjz * viy, wy = vjz * vix - vjx * viz,
                   wz = vjx * viy - vjy * vix;
      // R x (crr vi - G2 a2 - 2 G3 b1) - G2 dj x vi + 2 G2 X - 2 G3 (vj x vi)
      {
        const double ux_ = crr * vix - G[2] * a2x - g3 * b1x;
        const double uy_ = crr * viy - G[2] * a2y - g3 * b1y;
        const double uz_ = crr * viz - G[2] * a2z - g3 * b1z;
        const double qx = (y * uz_ - z * uy_) - G[2] * (djy * viz - djz * viy) + g2 * Xx - g3 * wx;
        const double qy = (z * ux_ - x * uz_) - G[2] * (djz * vix - djx * viz) + g2 * Xy - g3 * wy;
        const double qz = (x * uy_ - y * ux_) - G[2] * (djx * viy - djy * vix) + g2 * Xz - g3 * wz;
        tx += 2.0 * qx;
        ty += 2.0 * qy;
        tz += 2.0 * qz;
      }
      if (jside) {
        // partner j: same formulas with (qi, di, Qi) <-> (qj, dj, Qj), R -> -R
        const double c1j = G[1] * qi - G[2] * dir + G[3] * qir;
        const double hx = G[1] * dix - 2.0 * G[2] * vix + c1j * x;
        const double hy = G[1] * diy - 2.0 * G[2] * viy + c1j * y;
        const double hz = G[1] * diz - 2.0 * G[2] * viz + c1j * z;
        double ux = hy * djz - hz * djy;
        double uy = hz * djx - hx * djz;
        double uz = hx * djy - hy * djx;
        // tau_j/2 = crj R x vj + G2 (R x Qj di + di x vj) - 2 G2 X
        //           - 2 G3 (vi x vj + R x Qj vi)
        const double crj = G[2] * qi - G[3] * dir + G[4] * qir;
        const double ux_ = crj * vjx + G[2] * a1x - g3 * b2x;
        const double uy_ = crj * vjy + G[2] * a1y - g3 * b2y;
        const double uz_ = crj * vjz + G[2] * a1z - g3 * b2z;
        ux += 2.0 * ((y * uz_ - z * uy_) + G[2] * (diy * vjz - diz * vjy) - g2 * Xx + g3 * wx);
        uy += 2.0 * ((z * ux_ - x * uz_) + G[2] * (diz * vjx - dix * vjz) - g2 * Xy + g3 * wy);
        uz += 2.0 * ((x * uy_ - y * ux_) + G[2] * (dix * vjy - diy * vjx) - g2 * Xz + g3 * wz);
        atomicAdd(&a.force[j].x, gx);
        atomicAdd(&a.force[j].y, gy);
        atomicAdd(&a.force[j].z, gz);
        atomicAdd(&a.torque[j].x, ux);
        atomicAdd(&a.torque[j].y, uy);
        atomicAdd(&a.torque[j].z, uz);
      }
    };
    // half rows: a sorted row's pairs with j > i are its suffix
    const int start = (HALF && a.L.sorted) ? row_suffix(row, cnt, i, lane) : 0;
    run_row<false, PRUNED>(  // pruned rows: every slot in range, no compaction
        row + start, cnt - start, lane, a.pos, nullptr, ring,
        [&](int32_t& raw, const double4& pj, int32_t, double& x, double& y, double& z) {
          const int32_t j = raw & 0x7fffffff;
          const double r2 = min_image(a.b, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, x, y, z);
          const bool keep = PRUNED ? !(EXCL && raw < 0)  // same molecule (flag bit)
                                   : (r2 <= a.c2) && !(EXCL && same_group(pj, pi));
          raw = j;
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
      if (HALF) {  // force / torque were zeroed or hold the accumulated base
        atomicAdd(&a.force[i].x, fx);
        atomicAdd(&a.force[i].y, fy);
        atomicAdd(&a.force[i].z, fz);
        atomicAdd(&a.torque[i].x, tx);
        atomicAdd(&a.torque[i].y, ty);
        atomicAdd(&a.torque[i].z, tz);
      } else {
        if (a.accumulate) {
          const double4 f0 = a.force[i];
          fx += f0.x;
          fy += f0.y;
          fz += f0.z;
        }
        a.force[i] = make_double4(fx, fy, fz, 0.0);
        a.torque[i] = make_double4(tx, ty, tz, 0.0);
      }
    }
  }
  block_store_partials<10>(acc, a.partials);
}

template <bool PRUNED>
static void launch_mpole(mdg_ctx* c, MKArgs& k, bool ex) {
  if (c->deterministic) {
    if (ex) MDG_LAUNCH_SITES(c, "mpole", k.n_i, k, (k_mpole<true, PRUNED, false>));
    else MDG_LAUNCH_SITES(c, "mpole", k.n_i, k, (k_mpole<false, PRUNED, false>));
    finalize_partials(c, c->last_grid, 10, 10, 0.5);
    return;
  }
  const size_t bytes = (size_t)k.n_i * sizeof(double4);
  if (!k.accumulate) MDG_CUDA_CHECK(cudaMemsetAsync(k.force, 0, bytes, c->stream));
  MDG_CUDA_CHECK(cudaMemsetAsync(k.torque, 0, bytes, c->stream));
  if (ex) MDG_LAUNCH_SITES(c, "mpole", k.n_i, k, (k_mpole<true, PRUNED, true>));
  else MDG_LAUNCH_SITES(c, "mpole", k.n_i, k, (k_mpole<false, PRUNED, true>));
  finalize_partials(c, c->last_grid, 10, 10, 1.0);
}

void run_mpole(mdg_ctx* c, int list_id, double alpha, double cutoff, double electric,
               int exclude, bool accumulate) {
  const DevList& L = c->lists[list_id];
  MKArgs k;
  k.n_i = c->n_own;
  k.pos = c->pos;
  k.mp = c->mp;
  k.pq4 = c->pq4;
  k.mol = c->mol;
  k.L = kernel_rows(c, list_id, cutoff);
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = cutoff * cutoff;
  k.alpha = alpha;
  k.electric = electric;
  k.force = c->force;
  k.torque = c->torque;
  k.accumulate = accumulate ? 1 : 0;
  launch_mpole<false>(c, k, exclude && c->has_mol);
}

void run_mpole_pruned(mdg_ctx* c, double alpha, double electric, int exclude, bool accumulate) {
  const PrunedList& P = c->plist;
  MKArgs k;
  k.n_i = c->n_own;
  k.pos = c->pos;
  k.mp = c->mp;
  k.pq4 = c->pq4;
  k.mol = c->mol;
  k.L = ListView{P.nbr, P.cnt, P.cap, P.sorted};
  k.b = make_box(c->lx, c->ly, c->lz);
  k.c2 = P.cutoff * P.cutoff;
  k.alpha = alpha;
  k.electric = electric;
  k.force = c->force;
  k.torque = c->torque;
  k.accumulate = accumulate ? 1 : 0;
  launch_mpole<true>(c, k, exclude && c->has_mol);
}

}  // namespace mdg
