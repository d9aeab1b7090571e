// TEST INFRASTRUCTURE ONLY -- CPU oracle (see oracle/README.md).
//
// Filtered predicates and constructions, restating
//   /root/reference/pkg/src/tetrefine/predicates.py:14-308  (filters + exact)
//   /root/reference/pkg/src/tetrefine/geometry.py:48-199     (constructions)
// The float filters use the same expressions and bounds as the reference;
// the exact fallbacks evaluate the same determinants on scaled big integers
// (exact.hpp), so every returned sign is the exact sign.
#pragma once
#include "exact.hpp"
#include <stdexcept>

namespace orc {

struct DegenerateTet : std::runtime_error { DegenerateTet(const char* m) : std::runtime_error(m) {} };
struct DegenerateTri : std::runtime_error { DegenerateTri(const char* m) : std::runtime_error(m) {} };

// predicates.py:16-34 -- epsilon = 2^-53
static const double kEps = 1.1102230246251565e-16;
static const double kCcwBound = (3.0 + 16.0 * kEps) * kEps;
static const double kIccBound = (10.0 + 96.0 * kEps) * kEps;
static const double kO3dBound = (7.0 + 56.0 * kEps) * kEps;
static const double kIspBound = (16.0 + 224.0 * kEps) * kEps;

struct ExactStats { long long o2d = 0, icc = 0, o3d = 0, isp = 0; };
inline ExactStats& exact_stats() { static ExactStats s; return s; }

inline int sgn(double x) { return x > 0 ? 1 : (x < 0 ? -1 : 0); }

inline int orient2d_exact(const double* a, const double* b, const double* c) {
  double xs[6] = {a[0], a[1], b[0], b[1], c[0], c[1]};
  BigInt v[6];
  scaled_ints(xs, 6, v);
  BigInt det = (v[2] - v[0]) * (v[5] - v[1]) - (v[3] - v[1]) * (v[4] - v[0]);
  return det.sign;
}

inline int incircle2d_exact(const double* a, const double* b, const double* c, const double* d) {
  double xs[8] = {a[0], a[1], b[0], b[1], c[0], c[1], d[0], d[1]};
  BigInt v[8];
  scaled_ints(xs, 8, v);
  BigInt r[3][3];
  for (int k = 0; k < 3; ++k) {
    BigInt px = v[2 * k] - v[6], py = v[2 * k + 1] - v[7];
    r[k][0] = px; r[k][1] = py; r[k][2] = px * px + py * py;
  }
  BigInt det = r[0][0] * (r[1][1] * r[2][2] - r[1][2] * r[2][1])
             - r[0][1] * (r[1][0] * r[2][2] - r[1][2] * r[2][0])
             + r[0][2] * (r[1][0] * r[2][1] - r[1][1] * r[2][0]);
  return det.sign;
}

inline int orient3d_exact(const double* a, const double* b, const double* c, const double* d) {
  double xs[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  BigInt v[12];
  scaled_ints(xs, 12, v);
  BigInt ux = v[3] - v[0], uy = v[4] - v[1], uz = v[5] - v[2];
  BigInt vx = v[6] - v[0], vy = v[7] - v[1], vz = v[8] - v[2];
  BigInt wx = v[9] - v[0], wy = v[10] - v[1], wz = v[11] - v[2];
  BigInt det = ux * (vy * wz - vz * wy) - uy * (vx * wz - vz * wx) + uz * (vx * wy - vy * wx);
  return det.sign;
}

inline int insphere_exact(const double* a, const double* b, const double* c, const double* d, const double* e) {
  double xs[15] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2],
                   d[0], d[1], d[2], e[0], e[1], e[2]};
  BigInt v[15];
  scaled_ints(xs, 15, v);
  BigInt r[4][4];
  for (int k = 0; k < 4; ++k) {
    BigInt px = v[3 * k] - v[12], py = v[3 * k + 1] - v[13], pz = v[3 * k + 2] - v[14];
    r[k][0] = px; r[k][1] = py; r[k][2] = pz; r[k][3] = px * px + py * py + pz * pz;
  }
  auto det3 = [&](int i0, int i1, int i2) {
    const BigInt* r0 = r[i0]; const BigInt* r1 = r[i1]; const BigInt* r2 = r[i2];
    return r0[0] * (r1[1] * r2[2] - r1[2] * r2[1]) - r0[1] * (r1[0] * r2[2] - r1[2] * r2[0])
         + r0[2] * (r1[0] * r2[1] - r1[1] * r2[0]);
  };
  BigInt det = (-r[0][3]) * det3(1, 2, 3) + r[1][3] * det3(0, 2, 3) - r[2][3] * det3(0, 1, 3)
             + r[3][3] * det3(0, 1, 2);
  return -det.sign;
}

inline int orient2d(const double* a, const double* b, const double* c) {
  double detleft = (b[0] - a[0]) * (c[1] - a[1]);
  double detright = (b[1] - a[1]) * (c[0] - a[0]);
  double det = detleft - detright;
  double detsum = std::fabs(detleft) + std::fabs(detright);
  if (std::fabs(det) > kCcwBound * detsum) return sgn(det);
  exact_stats().o2d++;
  return orient2d_exact(a, b, c);
}

inline int incircle2d(const double* a, const double* b, const double* c, const double* d) {
  double adx = a[0] - d[0], ady = a[1] - d[1];
  double bdx = b[0] - d[0], bdy = b[1] - d[1];
  double cdx = c[0] - d[0], cdy = c[1] - d[1];
  double alift = adx * adx + ady * ady;
  double blift = bdx * bdx + bdy * bdy;
  double clift = cdx * cdx + cdy * cdy;
  double bxcy = bdx * cdy, bycx = bdy * cdx;
  double cxay = cdx * ady, cyax = cdy * adx;
  double axby = adx * bdy, aybx = ady * bdx;
  double det = alift * (bxcy - bycx) + blift * (cxay - cyax) + clift * (axby - aybx);
  double perm = alift * (std::fabs(bxcy) + std::fabs(bycx)) + blift * (std::fabs(cxay) + std::fabs(cyax))
              + clift * (std::fabs(axby) + std::fabs(aybx));
  if (std::fabs(det) > kIccBound * perm) return sgn(det);
  exact_stats().icc++;
  return incircle2d_exact(a, b, c, d);
}

inline int orient3d(const double* a, const double* b, const double* c, const double* d) {
  double adx = a[0] - d[0], ady = a[1] - d[1], adz = a[2] - d[2];
  double bdx = b[0] - d[0], bdy = b[1] - d[1], bdz = b[2] - d[2];
  double cdx = c[0] - d[0], cdy = c[1] - d[1], cdz = c[2] - d[2];
  double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  double cdxady = cdx * ady, adxcdy = adx * cdy;
  double adxbdy = adx * bdy, bdxady = bdx * ady;
  double det = adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  double perm = std::fabs(adz) * (std::fabs(bdxcdy) + std::fabs(cdxbdy))
              + std::fabs(bdz) * (std::fabs(cdxady) + std::fabs(adxcdy))
              + std::fabs(cdz) * (std::fabs(adxbdy) + std::fabs(bdxady));
  if (std::fabs(det) > kO3dBound * perm) return -sgn(det);
  exact_stats().o3d++;
  return orient3d_exact(a, b, c, d);
}

inline int insphere(const double* a, const double* b, const double* c, const double* d, const double* e) {
  double aex = a[0] - e[0], aey = a[1] - e[1], aez = a[2] - e[2];
  double bex = b[0] - e[0], bey = b[1] - e[1], bez = b[2] - e[2];
  double cex = c[0] - e[0], cey = c[1] - e[1], cez = c[2] - e[2];
  double dex = d[0] - e[0], dey = d[1] - e[1], dez = d[2] - e[2];
  double aexbey = aex * bey, bexaey = bex * aey, ab = aexbey - bexaey;
  double bexcey = bex * cey, cexbey = cex * bey, bc = bexcey - cexbey;
  double cexdey = cex * dey, dexcey = dex * cey, cd = cexdey - dexcey;
  double dexaey = dex * aey, aexdey = aex * dey, da = dexaey - aexdey;
  double aexcey = aex * cey, cexaey = cex * aey, ac = aexcey - cexaey;
  double bexdey = bex * dey, dexbey = dex * bey, bd = bexdey - dexbey;
  double abc = aez * bc - bez * ac + cez * ab;
  double bcd = bez * cd - cez * bd + dez * bc;
  double cda = cez * da + dez * ac + aez * cd;
  double dab = dez * ab + aez * bd + bez * da;
  double alift = aex * aex + aey * aey + aez * aez;
  double blift = bex * bex + bey * bey + bez * bez;
  double clift = cex * cex + cey * cey + cez * cez;
  double dlift = dex * dex + dey * dey + dez * dez;
  double det = (dlift * abc - clift * dab) + (blift * cda - alift * bcd);
  double aezp = std::fabs(aez), bezp = std::fabs(bez), cezp = std::fabs(cez), dezp = std::fabs(dez);
  double aexbeyp = std::fabs(aexbey), bexaeyp = std::fabs(bexaey);
  double bexceyp = std::fabs(bexcey), cexbeyp = std::fabs(cexbey);
  double cexdeyp = std::fabs(cexdey), dexceyp = std::fabs(dexcey);
  double dexaeyp = std::fabs(dexaey), aexdeyp = std::fabs(aexdey);
  double aexceyp = std::fabs(aexcey), cexaeyp = std::fabs(cexaey);
  double bexdeyp = std::fabs(bexdey), dexbeyp = std::fabs(dexbey);
  double perm = (((cexdeyp + dexceyp) * bezp + (dexbeyp + bexdeyp) * cezp + (bexceyp + cexbeyp) * dezp) * alift
               + ((dexaeyp + aexdeyp) * cezp + (aexceyp + cexaeyp) * dezp + (cexdeyp + dexceyp) * aezp) * blift
               + ((aexbeyp + bexaeyp) * dezp + (bexaeyp + aexbeyp) * aezp + (dexaeyp + aexdeyp) * bezp) * clift
               + ((bexceyp + cexbeyp) * aezp + (cexaeyp + aexceyp) * bezp + (aexbeyp + bexaeyp) * cezp) * dlift);
  if (std::fabs(det) > kIspBound * perm) return -sgn(det);
  exact_stats().isp++;
  return insphere_exact(a, b, c, d, e);
}

// predicates.py:286-308; raises on a degenerate triangle
inline int incircle3d(const double* a, const double* b, const double* c, const double* p) {
  double ux = b[0] - a[0], uy = b[1] - a[1], uz = b[2] - a[2];
  double vx = c[0] - a[0], vy = c[1] - a[1], vz = c[2] - a[2];
  double n[3] = {uy * vz - uz * vy, uz * vx - ux * vz, ux * vy - uy * vx};
  int order[3] = {0, 1, 2};
  // stable sort by -|n_k|
  std::stable_sort(order, order + 3, [&](int i, int j) { return std::fabs(n[i]) > std::fabs(n[j]); });
  for (int t = 0; t < 3; ++t) {
    int axis = order[t];
    int i = axis == 0 ? 1 : 0, j = axis == 2 ? 1 : 2;
    double a2[2] = {a[i], a[j]}, b2[2] = {b[i], b[j]}, c2[2] = {c[i], c[j]}, p2[2] = {p[i], p[j]};
    int s = orient2d(a2, b2, c2);
    if (s != 0) return s * incircle2d(a2, b2, c2, p2);
  }
  throw DegenerateTri("degenerate triangle in incircle3d");
}

struct Sphere { double c[3]; double r2; };

// geometry.py:74-98
inline Sphere circumsphere_tet_exact(const double* a, const double* b, const double* c, const double* d) {
  double xs[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  BigInt v[12];
  int ex = scaled_ints_exp(xs, 12, v);
  BigInt u[3], w1[3], w2[3];
  for (int k = 0; k < 3; ++k) { u[k] = v[3 + k] - v[k]; w1[k] = v[6 + k] - v[k]; w2[k] = v[9 + k] - v[k]; }
  // u, v=w1, w=w2
  BigInt vw[3] = {w1[1] * w2[2] - w1[2] * w2[1], w1[2] * w2[0] - w1[0] * w2[2], w1[0] * w2[1] - w1[1] * w2[0]};
  BigInt wu[3] = {w2[1] * u[2] - w2[2] * u[1], w2[2] * u[0] - w2[0] * u[2], w2[0] * u[1] - w2[1] * u[0]};
  BigInt uv[3] = {u[1] * w1[2] - u[2] * w1[1], u[2] * w1[0] - u[0] * w1[2], u[0] * w1[1] - u[1] * w1[0]};
  BigInt den = (u[0] * vw[0] + u[1] * vw[1] + u[2] * vw[2]) * BigInt(2);
  BigInt lu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  BigInt lv = w1[0] * w1[0] + w1[1] * w1[1] + w1[2] * w1[2];
  BigInt lw = w2[0] * w2[0] + w2[1] * w2[1] + w2[2] * w2[2];
  // off_k = N_k / den in scaled units (value = N_k/den * 2^ex)
  Sphere s;
  BigInt N[3];
  for (int k = 0; k < 3; ++k) N[k] = lu * vw[k] + lv * wu[k] + lw * uv[k];
  for (int k = 0; k < 3; ++k) {
    // centre = a + off = (a_S*den + N)/den * 2^ex
    BigInt num = v[k] * den + N[k];
    s.c[k] = rat_to_double(num, den, ex);
  }
  BigInt r2n = N[0] * N[0] + N[1] * N[1] + N[2] * N[2];
  s.r2 = rat_to_double(r2n, den * den, 2 * (int64_t)ex);
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(s.c[k])) throw DegenerateTet("circumcenter overflows float range");
  if (!std::isfinite(s.r2)) throw DegenerateTet("circumcenter overflows float range");
  return s;
}

// geometry.py:48-71
inline Sphere circumsphere_tet(const double* a, const double* b, const double* c, const double* d) {
  double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  double vw[3] = {v[1] * w[2] - v[2] * w[1], v[2] * w[0] - v[0] * w[2], v[0] * w[1] - v[1] * w[0]};
  double denom = 2.0 * (u[0] * vw[0] + u[1] * vw[1] + u[2] * vw[2]);
  if (denom == 0.0 || !std::isfinite(denom)) {
    if (orient3d(a, b, c, d) == 0) throw DegenerateTet("coplanar vertices");
    return circumsphere_tet_exact(a, b, c, d);
  }
  double lu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  double lv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  double lw = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  double wu[3] = {w[1] * u[2] - w[2] * u[1], w[2] * u[0] - w[0] * u[2], w[0] * u[1] - w[1] * u[0]};
  double uv[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  double ox = (lu * vw[0] + lv * wu[0] + lw * uv[0]) / denom;
  double oy = (lu * vw[1] + lv * wu[1] + lw * uv[1]) / denom;
  double oz = (lu * vw[2] + lv * wu[2] + lw * uv[2]) / denom;
  Sphere s;
  s.c[0] = a[0] + ox; s.c[1] = a[1] + oy; s.c[2] = a[2] + oz;
  s.r2 = ox * ox + oy * oy + oz * oz;
  return s;
}

// geometry.py:101-120
inline Sphere circumcircle_tri(const double* a, const double* b, const double* c) {
  double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  double nn = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
  if (nn == 0.0) throw DegenerateTri("collinear vertices");
  double lu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  double lv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  double q[3] = {lu * v[0] - lv * u[0], lu * v[1] - lv * u[1], lu * v[2] - lv * u[2]};
  double t[3] = {q[1] * n[2] - q[2] * n[1], q[2] * n[0] - q[0] * n[2], q[0] * n[1] - q[1] * n[0]};
  double ox = t[0] / (2.0 * nn), oy = t[1] / (2.0 * nn), oz = t[2] / (2.0 * nn);
  Sphere s;
  s.c[0] = a[0] + ox; s.c[1] = a[1] + oy; s.c[2] = a[2] + oz;
  s.r2 = ox * ox + oy * oy + oz * oz;
  return s;
}

inline double dist_sq(const double* a, const double* b) {
  double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

// geometry.py:132-156 (open diametral ball)
inline bool encroaches_segment(const double* u, const double* v, const double* p) {
  double f = 0.0, ssq = 0.0;
  for (int k = 0; k < 3; ++k) {
    double t = 2.0 * p[k] - u[k] - v[k];
    double e = u[k] - v[k];
    f += t * t - e * e;
    ssq += t * t + e * e;
  }
  if (std::fabs(f) > 1e-12 * ssq) return f < 0.0;
  double xs[9] = {p[0], p[1], p[2], u[0], u[1], u[2], v[0], v[1], v[2]};
  BigInt s[9];
  scaled_ints(xs, 9, s);
  BigInt total;
  for (int k = 0; k < 3; ++k) {
    BigInt t = s[k] * BigInt(2) - s[3 + k] - s[6 + k];
    BigInt e = s[3 + k] - s[6 + k];
    total = total + t * t - e * e;
  }
  return total.sign < 0;
}

// geometry.py:159-194: sign of |p-o|^2 - r^2 for the equatorial sphere
inline int equatorial_cmp(const double* a, const double* b, const double* c, const double* p) {
  Sphere sph = circumcircle_tri(a, b, c);
  double f = dist_sq(p, sph.c) - sph.r2;
  double scale = dist_sq(p, sph.c) + sph.r2;
  if (std::fabs(f) > 1e-9 * scale) return f > 0 ? 1 : -1;
  double xs[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], p[0], p[1], p[2]};
  BigInt s[12];
  scaled_ints(xs, 12, s);
  BigInt u[3], v[3], w[3];
  for (int k = 0; k < 3; ++k) { u[k] = s[3 + k] - s[k]; v[k] = s[6 + k] - s[k]; w[k] = s[9 + k] - s[k]; }
  BigInt uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  BigInt vv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  BigInt uv = u[0] * v[0] + u[1] * v[1] + u[2] * v[2];
  BigInt det = uu * vv - uv * uv;
  if (det.sign == 0) throw DegenerateTri("collinear vertices");
  // centre = a + x u + y v, x = (uu vv - uv vv)/(2 det), y = (vv uu - uv uu)/(2 det)
  // d2 - r2 = |w|^2 - 2 (x u.w + y v.w); times det > 0:
  BigInt ww = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  BigInt uw = u[0] * w[0] + u[1] * w[1] + u[2] * w[2];
  BigInt vw = v[0] * w[0] + v[1] * w[1] + v[2] * w[2];
  BigInt val = det * ww - (uu * vv - uv * vv) * uw - (vv * uu - uv * uu) * vw;
  return val.sign;
}

inline bool encroaches_face(const double* a, const double* b, const double* c, const double* p) {
  return equatorial_cmp(a, b, c, p) < 0;
}

}  // namespace orc
