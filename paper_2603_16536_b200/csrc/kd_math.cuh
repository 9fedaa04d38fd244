// kd_math.cuh — fp64 SE(3) primitives shared by host (model build) and device
// (per-step kernels).  Formulas follow the reference se3.cpp and the Eigen
// operations it relies on (Quaternion product / toRotationMatrix /
// Quaternion(Mat3) / q*v), SURVEY.md Appendix A.
#pragma once

#include <math.h>

#ifdef __CUDACC__
#define KD_HD __host__ __device__ __forceinline__
#else
#define KD_HD inline
#endif

namespace kd {

struct V3 {
  double x, y, z;
};
struct M3 {
  double m[9];  // row-major
};
struct Q4 {
  double w, x, y, z;
};

KD_HD V3 v3(double a, double b, double c) { return V3{a, b, c}; }
KD_HD V3 add(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
KD_HD V3 sub(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
KD_HD V3 neg(V3 a) { return V3{-a.x, -a.y, -a.z}; }
KD_HD V3 scl(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
KD_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
KD_HD double norm(V3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
KD_HD V3 cross(V3 a, V3 b) { return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
KD_HD double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

KD_HD M3 mzero() { return M3{{0, 0, 0, 0, 0, 0, 0, 0, 0}}; }
KD_HD M3 mident() { return M3{{1, 0, 0, 0, 1, 0, 0, 0, 1}}; }
KD_HD M3 mmul(const M3& a, const M3& b) {
  M3 o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double s = a.m[3 * r] * b.m[c];
      s += a.m[3 * r + 1] * b.m[3 + c];
      s += a.m[3 * r + 2] * b.m[6 + c];
      o.m[3 * r + c] = s;
    }
  return o;
}
KD_HD V3 mvec(const M3& a, V3 v) {
  return V3{a.m[0] * v.x + a.m[1] * v.y + a.m[2] * v.z, a.m[3] * v.x + a.m[4] * v.y + a.m[5] * v.z,
            a.m[6] * v.x + a.m[7] * v.y + a.m[8] * v.z};
}
// v^T A (row vector times matrix)
KD_HD V3 vmat(V3 v, const M3& a) {
  return V3{v.x * a.m[0] + v.y * a.m[3] + v.z * a.m[6], v.x * a.m[1] + v.y * a.m[4] + v.z * a.m[7],
            v.x * a.m[2] + v.y * a.m[5] + v.z * a.m[8]};
}
// A^T v
KD_HD V3 mtvec(const M3& a, V3 v) { return vmat(v, a); }
KD_HD M3 mtrans(const M3& a) {
  return M3{{a.m[0], a.m[3], a.m[6], a.m[1], a.m[4], a.m[7], a.m[2], a.m[5], a.m[8]}};
}
KD_HD M3 madd(const M3& a, const M3& b) {
  M3 o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] + b.m[i];
  return o;
}
KD_HD M3 msub(const M3& a, const M3& b) {
  M3 o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] - b.m[i];
  return o;
}
KD_HD M3 mscl(double s, const M3& a) {
  M3 o;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.m[i] = s * a.m[i];
  return o;
}
KD_HD V3 mrow(const M3& a, int r) { return V3{a.m[3 * r], a.m[3 * r + 1], a.m[3 * r + 2]}; }
KD_HD V3 mcol(const M3& a, int c) { return V3{a.m[c], a.m[3 + c], a.m[6 + c]}; }

// skew (se3.cpp:7-11)
KD_HD M3 skew(V3 v) { return M3{{0, -v.z, v.y, v.z, 0, -v.x, -v.y, v.x, 0}}; }

// Eigen Quaternion product
KD_HD Q4 qmul(Q4 a, Q4 b) {
  return Q4{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z, a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}
KD_HD double qnorm(Q4 q) { return sqrt(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w); }
KD_HD Q4 qnormalized(Q4 q) {
  const double n = qnorm(q);
  return Q4{q.w / n, q.x / n, q.y / n, q.z / n};
}
// Eigen toRotationMatrix
KD_HD M3 qrot(Q4 q) {
  const double tx = 2 * q.x, ty = 2 * q.y, tz = 2 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  return M3{{1 - (tyy + tzz), txy - twz, txz + twy, txy + twz, 1 - (txx + tzz), tyz - twx, txz - twy, tyz + twx,
             1 - (txx + tyy)}};
}
// Eigen Quaternion(Mat3)
KD_HD Q4 qfrom(const M3& m) {
  Q4 q;
  double t = m.m[0] + m.m[4] + m.m[8];
  if (t > 0) {
    t = sqrt(t + 1.0);
    q.w = 0.5 * t;
    t = 0.5 / t;
    q.x = (m.m[7] - m.m[5]) * t;
    q.y = (m.m[2] - m.m[6]) * t;
    q.z = (m.m[3] - m.m[1]) * t;
  } else {
    int i = 0;
    if (m.m[4] > m.m[0]) i = 1;
    if (m.m[8] > m.m[4 * i]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = sqrt(m.m[4 * i] - m.m[4 * j] - m.m[4 * k] + 1.0);
    double c[3];
    c[i] = 0.5 * t;
    t = 0.5 / t;
    q.w = (m.m[3 * k + j] - m.m[3 * j + k]) * t;
    c[j] = (m.m[3 * j + i] + m.m[3 * i + j]) * t;
    c[k] = (m.m[3 * k + i] + m.m[3 * i + k]) * t;
    q.x = c[0];
    q.y = c[1];
    q.z = c[2];
  }
  return q;
}
// Eigen q * v
KD_HD V3 qapply(Q4 q, V3 v) {
  const V3 qv{q.x, q.y, q.z};
  V3 uv = cross(qv, v);
  uv = add(uv, uv);
  return add(add(v, scl(q.w, uv)), cross(qv, uv));
}

// quat_exp (se3.cpp:13-25)
KD_HD Q4 quat_exp(V3 v) {
  const double angle = norm(v);
  double sinc;
  if (angle < 1e-8) {
    sinc = 1.0 - angle * angle / 6.0;
  } else {
    sinc = sin(angle) / angle;
  }
  const V3 s = scl(sinc, v);
  return Q4{cos(angle), s.x, s.y, s.z};
}
// quat_integrate (se3.cpp:27-32)
KD_HD Q4 quat_integrate(Q4 q, V3 w, double dt) { return qnormalized(qmul(q, quat_exp(scl(0.5 * dt, w)))); }

// so3_log(Quat) (se3.cpp:48-59)
KD_HD V3 so3_log_q(Q4 qin) {
  Q4 q = qnormalized(qin);
  if (q.w < 0) q = Q4{-q.w, -q.x, -q.y, -q.z};
  const V3 vq{q.x, q.y, q.z};
  const double vn = norm(vq);
  const double angle = 2.0 * atan2(vn, q.w);
  if (vn < 1e-12) return scl(2.0, vq);
  return scl(angle / vn, vq);
}
KD_HD V3 so3_log(const M3& r) { return so3_log_q(qfrom(r)); }

// left_jacobian_inverse (se3.cpp:63-74)
KD_HD M3 left_jacobian_inverse(V3 phi) {
  const double angle = norm(phi);
  const M3 k = skew(phi);
  double c;
  if (angle < 1e-4) {
    c = 1.0 / 12.0 + angle * angle / 720.0;
  } else {
    c = 1.0 / (angle * angle) - (1.0 + cos(angle)) / (2.0 * angle * sin(angle));
  }
  return madd(msub(mident(), mscl(0.5, k)), mmul(mscl(c, k), k));
}

// world_inertia (se3.cpp:76-80)
KD_HD M3 world_inertia(const M3& ib, Q4 q) {
  const M3 r = qrot(q);
  const M3 iw = mmul(mmul(r, ib), mtrans(r));
  return mscl(0.5, madd(iw, mtrans(iw)));
}

// Mat3::llt().solve(Identity) (delassus.cpp:30)
KD_HD M3 llt_inverse3(const M3& a) {
  double l[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double x = a.m[4 * k];
    for (int j = 0; j < k; ++j) x -= l[k][j] * l[k][j];
    x = sqrt(x);
    l[k][k] = x;
    for (int i = k + 1; i < 3; ++i) {
      double s = a.m[3 * i + k];
      for (int j = 0; j < k; ++j) s -= l[i][j] * l[k][j];
      l[i][k] = s / x;
    }
  }
  M3 inv;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double y[3];
    for (int i = 0; i < 3; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) s -= l[i][j] * y[j];
      y[i] = s / l[i][i];
    }
    for (int i = 2; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < 3; ++j) s -= l[j][i] * inv.m[3 * j + c];
      inv.m[3 * i + c] = s / l[i][i];
    }
  }
  return inv;
}

// orthonormal_complement (se3.cpp:97-110)
KD_HD void orthonormal_complement(V3 axis, V3& b1, V3& b2) {
  int least = 0;
  if (fabs(axis.y) < fabs(axis.x)) least = 1;
  if (fabs(axis.z) < fabs(comp(axis, least))) least = 2;
  V3 e{least == 0 ? 1.0 : 0.0, least == 1 ? 1.0 : 0.0, least == 2 ? 1.0 : 0.0};
  const V3 d = sub(e, scl(dot(e, axis), axis));
  const double nd = norm(d);
  b1 = V3{d.x / nd, d.y / nd, d.z / nd};
  b2 = cross(axis, b1);
}

}  // namespace kd
