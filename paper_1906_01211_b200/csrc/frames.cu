// frames.cu -- local multipole frames: the multipoles are
// given in a per-site frame built from two neighbouring atoms, rotated to
// the global frame every step, and the torques the multipole kernels
// produce are turned into forces on the frame atoms. Frame types (Tinker's
// conventions; the water oxygen is a bisector site, the hydrogens z-then-x):
//   1 z-then-x: z = unit(u), x = unit(v - (v.z) z), y = z x x
//   2 bisector: z = unit(unit(u) + unit(v)), x, y as above
// with u = r_zatom - r_i, v = r_xatom - r_i (minimum image).
//
// Torque -> force: an infinitesimal frame rotation dtheta changes the
// energy by -tau . dtheta. With the axes' responses dz = dtheta x z,
// dx = dtheta x x, the rotation components along the local axes are
// dth_x = -y.dz, dth_y = x.dz, dth_z = y.dx, so
//   dE/du = -(-tau_x Jzu^T y + tau_y Jzu^T x + tau_z Jxu^T y)   (same for v)
// with Jzu = dz/du etc. (3x3, from the normalisations above), and
// F_zatom = -dE/du, F_xatom = -dE/dv, F_i = dE/du + dE/dv (net force 0).
// The oracle (oracle/frames.py) checks all of it by finite differences of
// the energy with the frames rebuilt at displaced positions.
#include "common.cuh"

namespace mdg {

struct M3 {
  double a[3][3];
};

__device__ __forceinline__ double3 d3(double x, double y, double z) { return make_double3(x, y, z); }
__device__ __forceinline__ double dot3(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double3 scale3(double3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double3 add3(double3 a, double3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ double3 sub3(double3 a, double3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double3 cross3(double3 a, double3 b) {
  return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double get(double3 v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : v.z); }

// P(e)/len = (I - e e^T) / len: derivative of unit(w) w.r.t. w, e = unit(w)
__device__ __forceinline__ M3 proj(double3 e, double len) {
  M3 m;
  const double il = 1.0 / len;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m.a[r][c] = ((r == c ? 1.0 : 0.0) - get(e, r) * get(e, c)) * il;
  return m;
}

__device__ __forceinline__ M3 mul(const M3& A, const M3& B) {
  M3 m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      m.a[r][c] = A.a[r][0] * B.a[0][c] + A.a[r][1] * B.a[1][c] + A.a[r][2] * B.a[2][c];
  return m;
}

// A^T v
__device__ __forceinline__ double3 tmul(const M3& A, double3 v) {
  return d3(A.a[0][0] * v.x + A.a[1][0] * v.y + A.a[2][0] * v.z,
            A.a[0][1] * v.x + A.a[1][1] * v.y + A.a[2][1] * v.z,
            A.a[0][2] * v.x + A.a[1][2] * v.y + A.a[2][2] * v.z);
}

struct Frame {
  double3 x, y, z;
  M3 jzu, jzv, jxu, jxv;  // dz/du, dz/dv, dx/du, dx/dv
};

__device__ Frame build_frame(int type, double3 u, double3 v, bool jac) {
  Frame f;
  const double lu = sqrt(dot3(u, u)), lv = sqrt(dot3(v, v));
  const double3 uh = scale3(u, 1.0 / lu), vh = scale3(v, 1.0 / lv);
  double3 s;
  double ls;
  if (type == 2) {
    s = add3(uh, vh);
    ls = sqrt(dot3(s, s));
    f.z = scale3(s, 1.0 / ls);
  } else {
    s = u;
    ls = lu;
    f.z = uh;
  }
  const double vz = dot3(v, f.z);
  const double3 w = sub3(v, scale3(f.z, vz));
  const double lw = sqrt(dot3(w, w));
  f.x = scale3(w, 1.0 / lw);
  f.y = cross3(f.z, f.x);
  if (!jac) return f;
  const M3 pz = proj(f.z, ls);
  if (type == 2) {
    f.jzu = mul(pz, proj(uh, lu));
    f.jzv = mul(pz, proj(vh, lv));
  } else {
    f.jzu = pz;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) f.jzv.a[r][c] = 0.0;
  }
  // w = v - z (z.v): dw/du = -(z v^T + (z.v) I) dz/du,
  //                  dw/dv = I - z z^T - (z v^T + (z.v) I) dz/dv
  M3 a;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a.a[r][c] = get(f.z, r) * get(v, c) + (r == c ? vz : 0.0);
  const M3 px = proj(f.x, lw);
  M3 dwu = mul(a, f.jzu), dwv = mul(a, f.jzv);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      dwu.a[r][c] = -dwu.a[r][c];
      dwv.a[r][c] = (r == c ? 1.0 : 0.0) - get(f.z, r) * get(f.z, c) - dwv.a[r][c];
    }
  f.jxu = mul(px, dwu);
  f.jxv = mul(px, dwv);
  return f;
}

__device__ __forceinline__ double3 min_image3(const Box& b, double4 a, double4 o) {
  double dx, dy, dz;
  min_image(b, a.x, a.y, a.z, o.x, o.y, o.z, dx, dy, dz);
  return d3(dx, dy, dz);  // a - o
}

// global multipoles from the local ones: mu = R mu_l, Q = R Q_l R^T,
// R = [x y z] (columns)
__global__ void k_rotpole(int64_t n, Box b, const double4* __restrict__ pos,
                          const int4* __restrict__ frame, const double4* __restrict__ ml,
                          double4* __restrict__ mp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 fr = frame[i];
  const double4 l0 = ml[3 * i], l1 = ml[3 * i + 1], l2 = ml[3 * i + 2];
  if (fr.x == 0) {
    mp[3 * i] = l0;
    mp[3 * i + 1] = l1;
    mp[3 * i + 2] = l2;
    return;
  }
  const double4 pi = pos[i];
  const Frame f = build_frame(fr.x, min_image3(b, pos[fr.y], pi), min_image3(b, pos[fr.z], pi), false);
  const double R[3][3] = {{f.x.x, f.y.x, f.z.x}, {f.x.y, f.y.y, f.z.y}, {f.x.z, f.y.z, f.z.z}};
  const double dl[3] = {l0.x, l0.y, l0.z};
  const double Q[3][3] = {{l0.w, l1.x, l1.y}, {l1.x, l1.z, l1.w}, {l1.y, l1.w, l2.x}};
  double d[3], RQ[3][3], G[3][3];
  for (int r = 0; r < 3; ++r) d[r] = R[r][0] * dl[0] + R[r][1] * dl[1] + R[r][2] * dl[2];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) RQ[r][c] = R[r][0] * Q[0][c] + R[r][1] * Q[1][c] + R[r][2] * Q[2][c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) G[r][c] = RQ[r][0] * R[c][0] + RQ[r][1] * R[c][1] + RQ[r][2] * R[c][2];
  mp[3 * i] = make_double4(d[0], d[1], d[2], G[0][0]);
  mp[3 * i + 1] = make_double4(G[0][1], G[0][2], G[1][1], G[1][2]);
  mp[3 * i + 2] = make_double4(G[2][2], 0.0, 0.0, 0.0);
}

// per owned site: forces on (i, zatom, xatom) from its torque
__global__ void k_frame_forces(int64_t n, Box b, const double4* __restrict__ pos,
                               const int4* __restrict__ frame, const double4* __restrict__ torque,
                               double4* __restrict__ fbuf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 fr = frame[i];
  if (fr.x == 0) {
    fbuf[3 * i] = fbuf[3 * i + 1] = fbuf[3 * i + 2] = make_double4(0, 0, 0, 0);
    return;
  }
  const double4 pi = pos[i];
  const Frame f = build_frame(fr.x, min_image3(b, pos[fr.y], pi), min_image3(b, pos[fr.z], pi), true);
  const double4 t4 = torque[i];
  const double3 t = d3(t4.x, t4.y, t4.z);
  const double tx = dot3(t, f.x), ty = dot3(t, f.y), tz = dot3(t, f.z);
  // dE/du, dE/dv
  const double3 gu = scale3(add3(add3(scale3(tmul(f.jzu, f.y), -tx), scale3(tmul(f.jzu, f.x), ty)),
                                 scale3(tmul(f.jxu, f.y), tz)), -1.0);
  const double3 gv = scale3(add3(add3(scale3(tmul(f.jzv, f.y), -tx), scale3(tmul(f.jzv, f.x), ty)),
                                 scale3(tmul(f.jxv, f.y), tz)), -1.0);
  const double3 fi = add3(gu, gv);
  fbuf[3 * i] = make_double4(fi.x, fi.y, fi.z, 0.0);
  fbuf[3 * i + 1] = make_double4(-gu.x, -gu.y, -gu.z, 0.0);  // zatom
  fbuf[3 * i + 2] = make_double4(-gv.x, -gv.y, -gv.z, 0.0);  // xatom
}

// per atom, fixed order: own frame force + every reference as z / x atom
__global__ void k_frame_gather(int64_t n, const int32_t* __restrict__ ref_start,
                               const int32_t* __restrict__ ref, const double4* __restrict__ fbuf,
                               double4* __restrict__ force) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  double4 f = force[a];
  const double4 own = fbuf[3 * a];
  f.x += own.x;
  f.y += own.y;
  f.z += own.z;
  for (int32_t k = ref_start[a]; k < ref_start[a + 1]; ++k) {
    const int32_t code = ref[k];  // 2 * site + role (0: zatom, 1: xatom)
    const double4 g = fbuf[3 * (code >> 1) + 1 + (code & 1)];
    f.x += g.x;
    f.y += g.y;
    f.z += g.z;
  }
  force[a] = f;
}

void rotate_multipoles(mdg_ctx* c) {
  if (!c->has_frames) return;
  MDG_LAUNCH(c, "rotpole", grid_for(c->n, 256), 256, 0, k_rotpole, c->n,
             make_box(c->lx, c->ly, c->lz), c->pos, c->frame, c->mploc, c->mp);
}

void frame_torques_to_forces(mdg_ctx* c) {
  if (!c->has_frames) return;
  const Box b = make_box(c->lx, c->ly, c->lz);
  MDG_LAUNCH(c, "frame_forces", grid_for(c->n_own, 256), 256, 0, k_frame_forces, c->n_own, b,
             c->pos, c->frame, c->torque, c->fbuf);
  MDG_LAUNCH(c, "frame_gather", grid_for(c->n_own, 256), 256, 0, k_frame_gather, c->n_own,
             c->fref_start, c->fref, c->fbuf, c->force);
}

}  // namespace mdg
