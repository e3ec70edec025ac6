/*
 * mdo_fast.c -- CPU BASELINE PORT (test/bench infrastructure only).
 *
 * Closed-form (Tinker-style) half-list CPU kernels for the parts of the
 * north-star path the reference does not implement: real-space multipole
 * Ewald energy/forces/torques and the Ewald + Thole multipole field. Used as
 * the "port" leg of bench.py's CPU baseline / --impl reference where the
 * reference (oracle/_ref) has no kernel, compiled with the reference's Vec
 * flags. Validated against the T-tensor oracle (mdo.c) in tests/test_oracle.py.
 * Same argument conventions as mdo.h (original order, d = r_i - r_j).
 */
#include <math.h>
#include <string.h>

#include "mdo.h"

static inline double w1(double d, double L, double iL, double hL) {
  double t = fma(-nearbyint(d * iL), L, d);
  return (t >= hL) ? t - L : t;
}

static inline void bn6(double r, double r2, double alpha, int nmax, double* bn) {
  const double ir2 = 1.0 / r2;
  bn[0] = erfc(alpha * r) / r;
  const double alsq2 = 2.0 * alpha * alpha;
  double alsq2n = alpha > 0 ? 1.0 / (1.7724538509055160273 * alpha) : 0.0;
  const double e = exp(-alpha * alpha * r2);
  for (int k = 1; k <= nmax; ++k) {
    alsq2n *= alsq2;
    bn[k] = ((double)(2 * k - 1) * bn[k - 1] + alsq2n * e) * ir2;
  }
}

typedef struct { double xx, xy, xz, yy, yz, zz; } q6;

static inline void qv(const q6* Q, const double* v, double* o) {
  o[0] = Q->xx * v[0] + Q->xy * v[1] + Q->xz * v[2];
  o[1] = Q->xy * v[0] + Q->yy * v[1] + Q->yz * v[2];
  o[2] = Q->xz * v[0] + Q->yz * v[1] + Q->zz * v[2];
}

static inline double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

static inline void load_q(const mdo_system* s, size_t i, q6* Q) {
  const double* q = s->quadrupole + 6 * i;
  Q->xx = q[0]; Q->xy = q[1]; Q->xz = q[2]; Q->yy = q[3]; Q->yz = q[4]; Q->zz = q[5];
}

/* torque from GQ (dU/dQ, symmetric) on a site with quadrupole Q:
 * tau = 2 (M_zy, M_xz, M_yx), M = Q GQ - GQ Q */
static inline void qtorque(const q6* Q, const q6* G, double* t) {
  const double Mzy = (Q->xz * G->xy + Q->yz * G->yy + Q->zz * G->yz) -
                     (G->xz * Q->xy + G->yz * Q->yy + G->zz * Q->yz);
  const double Mxz = (Q->xx * G->xz + Q->xy * G->yz + Q->xz * G->zz) -
                     (G->xx * Q->xz + G->xy * Q->yz + G->xz * Q->zz);
  const double Myx = (Q->xy * G->xx + Q->yy * G->xy + Q->yz * G->xz) -
                     (G->xy * Q->xx + G->yy * Q->xy + G->yz * Q->xz);
  t[0] += 2.0 * Mzy;
  t[1] += 2.0 * Mxz;
  t[2] += 2.0 * Myx;
}

/* GQ = c_rr R R^T + c_dr (d R^T + R d^T) + c_q Q + c_vr (R v^T + v R^T) */
static inline void make_gq(double crr, double cdr, const double* d, double cq, const q6* Q,
                           double cvr, const double* v, const double* R, q6* G) {
  G->xx = crr * R[0] * R[0] + cdr * 2 * d[0] * R[0] + cq * Q->xx + cvr * 2 * R[0] * v[0];
  G->yy = crr * R[1] * R[1] + cdr * 2 * d[1] * R[1] + cq * Q->yy + cvr * 2 * R[1] * v[1];
  G->zz = crr * R[2] * R[2] + cdr * 2 * d[2] * R[2] + cq * Q->zz + cvr * 2 * R[2] * v[2];
  G->xy = crr * R[0] * R[1] + cdr * (d[0] * R[1] + R[0] * d[1]) + cq * Q->xy +
          cvr * (R[0] * v[1] + v[0] * R[1]);
  G->xz = crr * R[0] * R[2] + cdr * (d[0] * R[2] + R[0] * d[2]) + cq * Q->xz +
          cvr * (R[0] * v[2] + v[0] * R[2]);
  G->yz = crr * R[1] * R[2] + cdr * (d[1] * R[2] + R[1] * d[2]) + cq * Q->yz +
          cvr * (R[1] * v[2] + v[1] * R[2]);
}

int mdf_mpole(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
              double electric, int exclude, double* f, double* torque, double* energy,
              double* virial9) {
  double w[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}; /* pair virial sum R_a F_b, F on i */
  const size_t n = s->n;
  memset(f, 0, 3 * n * sizeof(double));
  memset(torque, 0, 3 * n * sizeof(double));
  const double L[3] = {s->lx, s->ly, s->lz};
  const double iL[3] = {1.0 / s->lx, 1.0 / s->ly, 1.0 / s->lz};
  const double hL[3] = {0.5 * s->lx, 0.5 * s->ly, 0.5 * s->lz};
  const double c2 = cutoff * cutoff;
  double etot = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    const double qi = s->charge[i];
    const double* di = s->dipole + 3 * i;
    q6 Qi;
    load_q(s, i, &Qi);
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      if (exclude && s->molecule && s->molecule[i] == s->molecule[j]) continue;
      double R[3] = {w1(s->x[i] - s->x[j], L[0], iL[0], hL[0]),
                     w1(s->y[i] - s->y[j], L[1], iL[1], hL[1]),
                     w1(s->z[i] - s->z[j], L[2], iL[2], hL[2])};
      const double r2 = fma(R[0], R[0], fma(R[1], R[1], R[2] * R[2]));
      if (!(r2 <= c2)) continue;
      const double r = sqrt(r2);
      double G[6];
      bn6(r, r2, alpha, 5, G);
      for (int q = 0; q < 6; ++q) G[q] *= electric;
      const double qj = s->charge[j];
      const double* dj = s->dipole + 3 * j;
      q6 Qj;
      load_q(s, j, &Qj);
      double vi[3], vj[3];
      qv(&Qi, R, vi);
      qv(&Qj, R, vj);
      const double dir = dot3(di, R), djr = dot3(dj, R);
      const double qir = dot3(R, vi), qjr = dot3(R, vj);
      const double dij = dot3(di, dj), diqj = dot3(di, vj), djqi = dot3(dj, vi);
      const double qiqj = Qi.xx * Qj.xx + Qi.yy * Qj.yy + Qi.zz * Qj.zz +
                          2.0 * (Qi.xy * Qj.xy + Qi.xz * Qj.xz + Qi.yz * Qj.yz);
      const double qvv = dot3(vi, vj);
      const double C0 = qi * qj, C1 = qi * djr - qj * dir + dij;
      const double C2 = qi * qjr + qj * qir - dir * djr + 2.0 * (diqj - djqi + qiqj);
      const double C3 = -dir * qjr + qir * djr - 4.0 * qvv;
      const double C4 = qir * qjr;
      etot += C0 * G[0] + C1 * G[1] + C2 * G[2] + C3 * G[3] + C4 * G[4];
      double a1[3], a2[3], b1[3], b2[3];
      qv(&Qj, di, a1);
      qv(&Qi, dj, a2);
      qv(&Qi, vj, b1);
      qv(&Qj, vi, b2);
      const double sc = C0 * G[1] + C1 * G[2] + C2 * G[3] + C3 * G[4] + C4 * G[5];
      for (int a = 0; a < 3; ++a) {
        const double g = G[1] * (qi * dj[a] - qj * di[a]) +
                         G[2] * (2.0 * (qi * vj[a] + qj * vi[a]) - djr * di[a] - dir * dj[a] +
                                 2.0 * (a1[a] - a2[a])) +
                         G[3] * (-qjr * di[a] - 2.0 * dir * vj[a] + 2.0 * djr * vi[a] +
                                 qir * dj[a] - 4.0 * (b1[a] + b2[a])) +
                         G[4] * 2.0 * (qjr * vi[a] + qir * vj[a]) - sc * R[a];
        f[3 * i + a] -= g;
        f[3 * j + a] += g;
        for (int b = 0; b < 3; ++b) w[3 * b + a] -= R[b] * g;
      }
      /* torque on i: gmu_i = G1 dj + 2 G2 vj - R (G1 qj + G2 djr + G3 qjr) */
      {
        const double c1 = G[1] * qj + G[2] * djr + G[3] * qjr;
        double gm[3];
        for (int a = 0; a < 3; ++a) gm[a] = G[1] * dj[a] + 2.0 * G[2] * vj[a] - c1 * R[a];
        double* ti = torque + 3 * i;
        ti[0] += gm[1] * di[2] - gm[2] * di[1];
        ti[1] += gm[2] * di[0] - gm[0] * di[2];
        ti[2] += gm[0] * di[1] - gm[1] * di[0];
        q6 GQ;
        make_gq(G[2] * qj + G[3] * djr + G[4] * qjr, -G[2], dj, 2.0 * G[2], &Qj, -2.0 * G[3], vj,
                R, &GQ);
        qtorque(&Qi, &GQ, ti);
      }
      /* torque on j: U(i,j;R) = U(j,i;-R) */
      {
        const double c1 = -G[1] * qi + G[2] * dir - G[3] * qir; /* coefficient of -R */
        double gm[3];
        for (int a = 0; a < 3; ++a) gm[a] = G[1] * di[a] - 2.0 * G[2] * vi[a] - c1 * R[a];
        double* tj = torque + 3 * j;
        tj[0] += gm[1] * dj[2] - gm[2] * dj[1];
        tj[1] += gm[2] * dj[0] - gm[0] * dj[2];
        tj[2] += gm[0] * dj[1] - gm[1] * dj[0];
        q6 GQ;
        make_gq(G[2] * qi - G[3] * dir + G[4] * qir, G[2], di, 2.0 * G[2], &Qi, -2.0 * G[3], vi,
                R, &GQ);
        qtorque(&Qj, &GQ, tj);
      }
    }
  }
  *energy = etot;
  if (virial9) memcpy(virial9, w, sizeof w);
  return 0;
}

/* E at `at` from the multipole at `src`, R = r_at - r_src (sign s = +1), or
 * at src from at (R -> -R) */
int mdf_perm_field(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                   double thole_a, int exclude, double* e) {
  const size_t n = s->n;
  memset(e, 0, 3 * n * sizeof(double));
  const double L[3] = {s->lx, s->ly, s->lz};
  const double iL[3] = {1.0 / s->lx, 1.0 / s->ly, 1.0 / s->lz};
  const double hL[3] = {0.5 * s->lx, 0.5 * s->ly, 0.5 * s->lz};
  const double c2 = cutoff * cutoff;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    const double pdi = cbrt(sqrt(s->polarizability[i]));
    q6 Qi;
    load_q(s, i, &Qi);
    const double* di = s->dipole + 3 * i;
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      if (exclude && s->molecule && s->molecule[i] == s->molecule[j]) continue;
      double R[3] = {w1(s->x[i] - s->x[j], L[0], iL[0], hL[0]),
                     w1(s->y[i] - s->y[j], L[1], iL[1], hL[1]),
                     w1(s->z[i] - s->z[j], L[2], iL[2], hL[2])};
      const double r2 = fma(R[0], R[0], fma(R[1], R[1], R[2] * R[2]));
      if (!(r2 <= c2)) continue;
      const double r = sqrt(r2), ir2 = 1.0 / r2;
      double bn[4];
      bn6(r, r2, alpha, 3, bn);
      const double u = r / (pdi * cbrt(sqrt(s->polarizability[j])));
      const double au3 = thole_a * u * u * u, ex = exp(-au3);
      const double l3 = 1.0 - ex, l5 = 1.0 - (1.0 + au3) * ex,
                   l7 = 1.0 - (1.0 + au3 + 0.6 * au3 * au3) * ex;
      const double b1 = ir2 / r, b2 = 3.0 * b1 * ir2, b3 = 5.0 * b2 * ir2;
      const double rr3 = bn[1] - (1.0 - l3) * b1, rr5 = bn[2] - (1.0 - l5) * b2,
                   rr7 = bn[3] - (1.0 - l7) * b3;
      q6 Qj;
      load_q(s, j, &Qj);
      const double* dj = s->dipole + 3 * j;
      double vi[3], vj[3];
      qv(&Qi, R, vi);
      qv(&Qj, R, vj);
      const double cj = rr3 * s->charge[j] + rr5 * dot3(dj, R) + rr7 * dot3(R, vj);
      /* at j: R' = -R: QiR' = -vi, mu.R' = -dir, R'QR' = qir */
      const double ci = rr3 * s->charge[i] - rr5 * dot3(di, R) + rr7 * dot3(R, vi);
      for (int a = 0; a < 3; ++a) {
        e[3 * i + a] += cj * R[a] - rr3 * dj[a] - 2.0 * rr5 * vj[a];
        e[3 * j + a] += -ci * R[a] - rr3 * di[a] + 2.0 * rr5 * vi[a];
      }
    }
  }
  return 0;
}

/* Ewald + Thole T mat-vec, half list */
int mdf_tmatvec(const mdo_system* s, const mdo_table* t, double alpha, double cutoff,
                double thole_a, const double* mu, double* e) {
  const size_t n = s->n;
  memset(e, 0, 3 * n * sizeof(double));
  const double L[3] = {s->lx, s->ly, s->lz};
  const double iL[3] = {1.0 / s->lx, 1.0 / s->ly, 1.0 / s->lz};
  const double hL[3] = {0.5 * s->lx, 0.5 * s->ly, 0.5 * s->lz};
  const double c2 = cutoff * cutoff;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* idx = t->indices + t->offset[i];
    const double pdi = cbrt(sqrt(s->polarizability[i]));
    const double* mi = mu + 3 * i;
    double ei[3] = {0, 0, 0};
    for (uint32_t k = 0; k < t->nnvlst[i]; ++k) {
      const size_t j = (size_t)idx[k];
      double R[3] = {w1(s->x[i] - s->x[j], L[0], iL[0], hL[0]),
                     w1(s->y[i] - s->y[j], L[1], iL[1], hL[1]),
                     w1(s->z[i] - s->z[j], L[2], iL[2], hL[2])};
      const double r2 = fma(R[0], R[0], fma(R[1], R[1], R[2] * R[2]));
      if (!(r2 <= c2)) continue;
      const double r = sqrt(r2), ir2 = 1.0 / r2;
      double bn[3];
      bn6(r, r2, alpha, 2, bn);
      const double u = r / (pdi * cbrt(sqrt(s->polarizability[j])));
      const double au3 = thole_a * u * u * u, ex = exp(-au3);
      const double l3 = 1.0 - ex, l5 = 1.0 - (1.0 + au3) * ex;
      const double b1 = ir2 / r;
      const double rr3 = bn[1] - (1.0 - l3) * b1, rr5 = bn[2] - (1.0 - l5) * 3.0 * b1 * ir2;
      const double* mj = mu + 3 * j;
      const double dj = dot3(mj, R), di = dot3(mi, R);
      for (int a = 0; a < 3; ++a) {
        ei[a] += rr5 * dj * R[a] - rr3 * mj[a];
        e[3 * j + a] += rr5 * di * R[a] - rr3 * mi[a];
      }
    }
    for (int a = 0; a < 3; ++a) e[3 * i + a] += ei[a];
  }
  return 0;
}
