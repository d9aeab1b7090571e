// gq_exact.cuh -- exact-decision geometric predicates and constructions for
// sm_100a.
//
// Semantics follow /root/reference/pkg/src/tetrefine/predicates.py:14-308 and
// geometry.py:48-199: the same float filter expressions and error bounds
// decide the common case; when a filter cannot certify the sign, the sign is
// computed exactly on big integers obtained by scaling every coordinate to a
// common power of two (frexp mantissa << (exponent - min exponent)), exactly
// as the reference's exact path does.  The big integers are fixed-width
// (GQ_BI_LIMBS x 32 bit) and live in local memory; an input whose exponent
// spread would overflow them raises the device error flag (never silently).
//
// Compiled with -fmad=false: every float expression rounds like the
// reference's (no contraction), so constructions are bit-identical.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef GQ_BI_LIMBS
#define GQ_BI_LIMBS 30     // 960 bits (far circumcentres are pulled in first, make_cand)
#endif

namespace gq {

// device-wide error record: the bits ever raised (for the message) and a count
// of raises that is never reset.  A context takes the count at the start of a
// call and fails when it has grown: concurrent contexts (C5) never wipe or lose
// each other's errors (an error raised by one is also reported by the others
// running at that time; every error is fatal).
__device__ unsigned int g_err;
__device__ unsigned long long g_errn;
#define GQ_ERR_BIGINT 1u
#define GQ_ERR_DEGEN 2u
#define GQ_ERR_CAP 4u
#define GQ_ERR_HASH 8u
#define GQ_ERR_STAR 16u
#define GQ_ERR_WALK 32u
#define GQ_ERR_2D 64u
__device__ __forceinline__ void raise_err_(unsigned int e) { atomicOr(&g_err, e); atomicAdd(&g_errn, 1ull); }
#ifdef GQ_DEBUG2D
#define raise_err(e) do { printf("[err] %u at %s:%d\n", (unsigned)(e), __FILE__, __LINE__); raise_err_(e); } while (0)
#else
#define raise_err(e) raise_err_(e)
#endif

// exact-call counters (instrumentation for the roofline / report)
__device__ unsigned long long g_exact_calls[4];

struct BI {
  int s;   // sign -1/0/+1
  int n;   // used limbs
  uint32_t d[GQ_BI_LIMBS];
};

__device__ __forceinline__ void bi_zero(BI& a) { a.s = 0; a.n = 0; }
__device__ __forceinline__ void bi_trim(BI& a) {
  while (a.n > 0 && a.d[a.n - 1] == 0) --a.n;
  if (a.n == 0) a.s = 0;
}
// a = m * 2^sh (m signed 64-bit)
__device__ __noinline__ void bi_set(BI& a, long long m, int sh) {
  bi_zero(a);
  if (m == 0) return;
  a.s = m < 0 ? -1 : 1;
  unsigned long long u = m < 0 ? (unsigned long long)(-(m + 1)) + 1ull : (unsigned long long)m;
  int w = sh >> 5, b = sh & 31;
  if (w + 3 > GQ_BI_LIMBS) { raise_err(GQ_ERR_BIGINT); bi_zero(a); return; }
  for (int i = 0; i < w; ++i) a.d[i] = 0;
  unsigned long long lo = (u << b) & 0xffffffffull;
  unsigned long long mid = b ? ((u >> (32 - b)) & 0xffffffffull) : ((u >> 32) & 0xffffffffull);
  unsigned long long hi = b ? (u >> (64 - b)) : 0ull;
  a.d[w] = (uint32_t)lo;
  a.d[w + 1] = (uint32_t)mid;
  a.d[w + 2] = (uint32_t)hi;
  a.n = w + 3;
  bi_trim(a);
}
__device__ inline int bi_cmpmag(const BI& a, const BI& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
  return 0;
}
// r = |a| + |b| (sign s)
__device__ inline void bi_addmag(BI& r, const BI& a, const BI& b, int s) {
  int n = a.n > b.n ? a.n : b.n;
  unsigned long long c = 0;
  for (int i = 0; i < n; ++i) {
    unsigned long long t = c + (i < a.n ? a.d[i] : 0u) + (i < b.n ? b.d[i] : 0u);
    r.d[i] = (uint32_t)t;
    c = t >> 32;
  }
  r.n = n;
  if (c) {
    if (n >= GQ_BI_LIMBS) { raise_err(GQ_ERR_BIGINT); bi_zero(r); return; }
    r.d[n] = (uint32_t)c; r.n = n + 1;
  }
  r.s = s;
  bi_trim(r);
}
// r = |a| - |b| with |a| >= |b| (sign s)
__device__ inline void bi_submag(BI& r, const BI& a, const BI& b, int s) {
  long long br = 0;
  for (int i = 0; i < a.n; ++i) {
    long long t = (long long)a.d[i] - br - (i < b.n ? (long long)b.d[i] : 0ll);
    if (t < 0) { t += (1ll << 32); br = 1; } else br = 0;
    r.d[i] = (uint32_t)t;
  }
  r.n = a.n;
  r.s = s;
  bi_trim(r);
}
__device__ __noinline__ void bi_add(BI& r, const BI& a, const BI& b) {  // r may alias nothing
  if (a.s == 0) { r = b; return; }
  if (b.s == 0) { r = a; return; }
  if (a.s == b.s) { bi_addmag(r, a, b, a.s); return; }
  int c = bi_cmpmag(a, b);
  if (c == 0) { bi_zero(r); return; }
  if (c > 0) bi_submag(r, a, b, a.s); else bi_submag(r, b, a, b.s);
}
__device__ inline void bi_neg(BI& a) { a.s = -a.s; }
__device__ __noinline__ void bi_sub(BI& r, const BI& a, const BI& b) { BI nb = b; bi_neg(nb); bi_add(r, a, nb); }
__device__ __noinline__ void bi_mul(BI& r, const BI& a, const BI& b) {
  bi_zero(r);
  if (a.s == 0 || b.s == 0) return;
  int n = a.n + b.n;
  if (n > GQ_BI_LIMBS) { raise_err(GQ_ERR_BIGINT); return; }
  for (int i = 0; i < n; ++i) r.d[i] = 0;
  for (int i = 0; i < a.n; ++i) {
    unsigned long long c = 0;
    for (int j = 0; j < b.n; ++j) {
      unsigned long long t = (unsigned long long)a.d[i] * b.d[j] + r.d[i + j] + c;
      r.d[i + j] = (uint32_t)t;
      c = t >> 32;
    }
    int k = i + b.n;
    while (c && k < n) {
      unsigned long long t = (unsigned long long)r.d[k] + c;
      r.d[k] = (uint32_t)t;
      c = t >> 32;
      ++k;
    }
  }
  r.n = n;
  r.s = a.s * b.s;
  bi_trim(r);
}
__device__ inline void bi_mulsmall(BI& r, const BI& a, int k) { BI t; bi_set(t, k, 0); bi_mul(r, a, t); }

// scaled integers of n doubles (zeros contribute no exponent)
__device__ __noinline__ int scaled(const double* x, int n, BI* out) {
  int emin = 1 << 30;
  for (int i = 0; i < n; ++i) {
    if (x[i] != 0.0) { int e; frexp(x[i], &e); emin = e < emin ? e : emin; }
  }
  if (emin == (1 << 30)) emin = 0;
#ifdef GQ_DEBUG2D
  {
    int emax = -(1 << 30);
    for (int i = 0; i < n; ++i) if (x[i] != 0.0) { int e; frexp(x[i], &e); emax = e > emax ? e : emax; }
    if (emax - emin > 120) {
      printf("[bigspread] n %d spread %d:", n, emax - emin);
      for (int i = 0; i < n; ++i) printf(" %.17g", x[i]);
      printf("\n");
    }
  }
#endif
  for (int i = 0; i < n; ++i) {
    if (x[i] == 0.0) { bi_zero(out[i]); continue; }
    int e;
    double m = frexp(x[i], &e);
    long long mi = (long long)(m * 9007199254740992.0);
    bi_set(out[i], mi, e - emin);
  }
  return emin - 53;
}

// ---------------------------------------------------------------------------
// filter constants (predicates.py:16-34; epsilon = 2^-53)
#define GQ_EPS 1.1102230246251565e-16
#define GQ_CCW_BOUND ((3.0 + 16.0 * GQ_EPS) * GQ_EPS)
#define GQ_ICC_BOUND ((10.0 + 96.0 * GQ_EPS) * GQ_EPS)
#define GQ_O3D_BOUND ((7.0 + 56.0 * GQ_EPS) * GQ_EPS)
#define GQ_ISP_BOUND ((16.0 + 224.0 * GQ_EPS) * GQ_EPS)

__device__ __forceinline__ int fsign(double x) { return x > 0.0 ? 1 : (x < 0.0 ? -1 : 0); }

__device__ __noinline__ int orient2d_exact(const double* a, const double* b, const double* c) {
  double xs[6] = {a[0], a[1], b[0], b[1], c[0], c[1]};
  BI v[6];
  scaled(xs, 6, v);
  BI p, q, t1, t2, det;
  bi_sub(p, v[2], v[0]); bi_sub(q, v[5], v[1]); bi_mul(t1, p, q);
  bi_sub(p, v[3], v[1]); bi_sub(q, v[4], v[0]); bi_mul(t2, p, q);
  bi_sub(det, t1, t2);
  return det.s;
}

__device__ inline int orient2d(const double* a, const double* b, const double* c) {
  double detleft = (b[0] - a[0]) * (c[1] - a[1]);
  double detright = (b[1] - a[1]) * (c[0] - a[0]);
  double det = detleft - detright;
  double detsum = fabs(detleft) + fabs(detright);
  if (fabs(det) > GQ_CCW_BOUND * detsum) return fsign(det);
  atomicAdd(&g_exact_calls[0], 1ull);
  return orient2d_exact(a, b, c);
}

__device__ __noinline__ int incircle2d_exact(const double* a, const double* b, const double* c, const double* d) {
  double xs[8] = {a[0], a[1], b[0], b[1], c[0], c[1], d[0], d[1]};
  BI v[8];
  scaled(xs, 8, v);
  BI r[3][3];
  for (int k = 0; k < 3; ++k) {
    BI t1, t2;
    bi_sub(r[k][0], v[2 * k], v[6]);
    bi_sub(r[k][1], v[2 * k + 1], v[7]);
    bi_mul(t1, r[k][0], r[k][0]); bi_mul(t2, r[k][1], r[k][1]);
    bi_add(r[k][2], t1, t2);
  }
  BI m1, m2, d1, t, acc, acc2;
  // r00*(r11 r22 - r12 r21)
  bi_mul(m1, r[1][1], r[2][2]); bi_mul(m2, r[1][2], r[2][1]); bi_sub(d1, m1, m2); bi_mul(acc, r[0][0], d1);
  bi_mul(m1, r[1][0], r[2][2]); bi_mul(m2, r[1][2], r[2][0]); bi_sub(d1, m1, m2); bi_mul(t, r[0][1], d1);
  bi_sub(acc2, acc, t);
  bi_mul(m1, r[1][0], r[2][1]); bi_mul(m2, r[1][1], r[2][0]); bi_sub(d1, m1, m2); bi_mul(t, r[0][2], d1);
  bi_add(acc, acc2, t);
  return acc.s;
}

__device__ inline int incircle2d(const double* a, const double* b, const double* c, const double* d) {
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
  double perm = alift * (fabs(bxcy) + fabs(bycx)) + blift * (fabs(cxay) + fabs(cyax)) + clift * (fabs(axby) + fabs(aybx));
  if (fabs(det) > GQ_ICC_BOUND * perm) return fsign(det);
  atomicAdd(&g_exact_calls[1], 1ull);
  return incircle2d_exact(a, b, c, d);
}

__device__ __noinline__ int orient3d_exact(const double* a, const double* b, const double* c, const double* d) {
  // a shared coordinate plane makes the determinant exactly zero
  for (int k = 0; k < 3; ++k)
    if (a[k] == b[k] && a[k] == c[k] && a[k] == d[k]) return 0;
  double xs[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  BI v[12];
  scaled(xs, 12, v);
  BI u[3], w1[3], w2[3];
  for (int k = 0; k < 3; ++k) { bi_sub(u[k], v[3 + k], v[k]); bi_sub(w1[k], v[6 + k], v[k]); bi_sub(w2[k], v[9 + k], v[k]); }
  BI m1, m2, d1, t, acc, acc2;
  bi_mul(m1, w1[1], w2[2]); bi_mul(m2, w1[2], w2[1]); bi_sub(d1, m1, m2); bi_mul(acc, u[0], d1);
  bi_mul(m1, w1[0], w2[2]); bi_mul(m2, w1[2], w2[0]); bi_sub(d1, m1, m2); bi_mul(t, u[1], d1);
  bi_sub(acc2, acc, t);
  bi_mul(m1, w1[0], w2[1]); bi_mul(m2, w1[1], w2[0]); bi_sub(d1, m1, m2); bi_mul(t, u[2], d1);
  bi_add(acc, acc2, t);
  return acc.s;
}

__device__ inline int orient3d(const double* a, const double* b, const double* c, const double* d) {
  double adx = a[0] - d[0], ady = a[1] - d[1], adz = a[2] - d[2];
  double bdx = b[0] - d[0], bdy = b[1] - d[1], bdz = b[2] - d[2];
  double cdx = c[0] - d[0], cdy = c[1] - d[1], cdz = c[2] - d[2];
  double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  double cdxady = cdx * ady, adxcdy = adx * cdy;
  double adxbdy = adx * bdy, bdxady = bdx * ady;
  double det = adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  double perm = fabs(adz) * (fabs(bdxcdy) + fabs(cdxbdy)) + fabs(bdz) * (fabs(cdxady) + fabs(adxcdy))
              + fabs(cdz) * (fabs(adxbdy) + fabs(bdxady));
  if (fabs(det) > GQ_O3D_BOUND * perm) return -fsign(det);
  // four points on one axis-aligned plane (box and cube faces): exactly zero
  for (int k = 0; k < 3; ++k)
    if (a[k] == b[k] && a[k] == c[k] && a[k] == d[k]) return 0;
  atomicAdd(&g_exact_calls[2], 1ull);
  return orient3d_exact(a, b, c, d);
}

__device__ __noinline__ int insphere_exact(const double* a, const double* b, const double* c, const double* d, const double* e) {
  double xs[15] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2], e[0], e[1], e[2]};
  BI v[15];
  scaled(xs, 15, v);
  BI r[4][4];
  for (int k = 0; k < 4; ++k) {
    BI t1, t2, t3;
    bi_sub(r[k][0], v[3 * k], v[12]);
    bi_sub(r[k][1], v[3 * k + 1], v[13]);
    bi_sub(r[k][2], v[3 * k + 2], v[14]);
    bi_mul(t1, r[k][0], r[k][0]); bi_mul(t2, r[k][1], r[k][1]); bi_add(t3, t1, t2);
    bi_mul(t1, r[k][2], r[k][2]); bi_add(r[k][3], t3, t1);
  }
  // det3 over columns 0..2 of rows (i0,i1,i2)
  auto det3 = [&](BI& out, int i0, int i1, int i2) {
    BI m1, m2, d1, t, acc;
    bi_mul(m1, r[i1][1], r[i2][2]); bi_mul(m2, r[i1][2], r[i2][1]); bi_sub(d1, m1, m2); bi_mul(acc, r[i0][0], d1);
    bi_mul(m1, r[i1][0], r[i2][2]); bi_mul(m2, r[i1][2], r[i2][0]); bi_sub(d1, m1, m2); bi_mul(t, r[i0][1], d1);
    bi_sub(out, acc, t);
    bi_mul(m1, r[i1][0], r[i2][1]); bi_mul(m2, r[i1][1], r[i2][0]); bi_sub(d1, m1, m2); bi_mul(t, r[i0][2], d1);
    bi_add(acc, out, t);
    out = acc;
  };
  BI D, t, acc, acc2;
  det3(D, 1, 2, 3); bi_mul(acc, r[0][3], D); bi_neg(acc);
  det3(D, 0, 2, 3); bi_mul(t, r[1][3], D); bi_add(acc2, acc, t);
  det3(D, 0, 1, 3); bi_mul(t, r[2][3], D); bi_sub(acc, acc2, t);
  det3(D, 0, 1, 2); bi_mul(t, r[3][3], D); bi_add(acc2, acc, t);
  return -acc2.s;
}

__device__ inline int insphere(const double* a, const double* b, const double* c, const double* d, const double* e) {
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
  double aezp = fabs(aez), bezp = fabs(bez), cezp = fabs(cez), dezp = fabs(dez);
  double aexbeyp = fabs(aexbey), bexaeyp = fabs(bexaey), bexceyp = fabs(bexcey), cexbeyp = fabs(cexbey);
  double cexdeyp = fabs(cexdey), dexceyp = fabs(dexcey), dexaeyp = fabs(dexaey), aexdeyp = fabs(aexdey);
  double aexceyp = fabs(aexcey), cexaeyp = fabs(cexaey), bexdeyp = fabs(bexdey), dexbeyp = fabs(dexbey);
  double perm = (((cexdeyp + dexceyp) * bezp + (dexbeyp + bexdeyp) * cezp + (bexceyp + cexbeyp) * dezp) * alift
               + ((dexaeyp + aexdeyp) * cezp + (aexceyp + cexaeyp) * dezp + (cexdeyp + dexceyp) * aezp) * blift
               + ((aexbeyp + bexaeyp) * dezp + (bexaeyp + aexbeyp) * aezp + (dexaeyp + aexdeyp) * bezp) * clift
               + ((bexceyp + cexbeyp) * aezp + (cexaeyp + aexceyp) * bezp + (aexbeyp + bexaeyp) * cezp) * dlift);
  if (fabs(det) > GQ_ISP_BOUND * perm) return -fsign(det);
  atomicAdd(&g_exact_calls[3], 1ull);
  return insphere_exact(a, b, c, d, e);
}

// predicates.py:286-308 (stable dominant-axis order); degenerate -> error flag
__device__ __noinline__ int incircle3d(const double* a, const double* b, const double* c, const double* p) {
  double ux = b[0] - a[0], uy = b[1] - a[1], uz = b[2] - a[2];
  double vx = c[0] - a[0], vy = c[1] - a[1], vz = c[2] - a[2];
  double an[3] = {fabs(uy * vz - uz * vy), fabs(uz * vx - ux * vz), fabs(ux * vy - uy * vx)};
  int o[3] = {0, 1, 2};
  // stable sort descending by |n|
  if (an[o[1]] > an[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  if (an[o[2]] > an[o[1]]) { int t = o[1]; o[1] = o[2]; o[2] = t; }
  if (an[o[1]] > an[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  // the bubble above is not stable for equal keys only when swapping equal
  // values, which it never does (strict >), so ties keep index order
  for (int t = 0; t < 3; ++t) {
    int axis = o[t];
    int i = axis == 0 ? 1 : 0, j = axis == 2 ? 1 : 2;
    double a2[2] = {a[i], a[j]}, b2[2] = {b[i], b[j]}, c2[2] = {c[i], c[j]}, p2[2] = {p[i], p[j]};
    int s = orient2d(a2, b2, c2);
    if (s != 0) return s * incircle2d(a2, b2, c2, p2);
  }
  raise_err(GQ_ERR_DEGEN);
  return 0;
}

// ---------------------------------------------------------------------------
// exact rational -> double (round half even), value = num/den * 2^exp2
__device__ inline int bi_bitlen(const BI& a) {
  if (a.n == 0) return 0;
  uint32_t t = a.d[a.n - 1];
  return (a.n - 1) * 32 + (32 - __clz(t));
}
__device__ __noinline__ void bi_shl(BI& r, const BI& a, int bits) {
  if (a.s == 0) { bi_zero(r); return; }
  int w = bits >> 5, b = bits & 31;
  if (a.n + w + 1 > GQ_BI_LIMBS) { raise_err(GQ_ERR_BIGINT); bi_zero(r); return; }
  BI t;
  for (int i = 0; i < w; ++i) t.d[i] = 0;
  uint32_t carry = 0;
  for (int i = 0; i < a.n; ++i) {
    unsigned long long v = ((unsigned long long)a.d[i] << b) | carry;
    t.d[w + i] = (uint32_t)v;
    carry = b ? (uint32_t)(v >> 32) : 0;
  }
  t.n = a.n + w;
  if (carry) { t.d[t.n] = carry; t.n++; }
  t.s = a.s;
  bi_trim(t);
  r = t;
}
__device__ __noinline__ double rat_to_double(const BI& num, const BI& den, int exp2) {
  if (num.s == 0) return 0.0;
  int sgn = num.s * den.s;
  BI n = num; n.s = 1;
  BI d = den; d.s = 1;
  int k = 56 - (bi_bitlen(n) - bi_bitlen(d));
  BI nn, dd;
  if (k >= 0) { bi_shl(nn, n, k); dd = d; } else { nn = n; bi_shl(dd, d, -k); }
  int qbits = bi_bitlen(nn) - bi_bitlen(dd) + 1;
  unsigned long long q = 0;
  BI r = nn;
  for (int i = qbits - 1; i >= 0; --i) {
    BI t, diff;
    bi_shl(t, dd, i);
    q <<= 1;
    bi_sub(diff, r, t);
    if (diff.s >= 0) { r = diff; q |= 1ull; }
  }
  bool sticky = r.s != 0;
  long long e = (long long)exp2 - k;
  int qb = 64 - __clzll(q);
  long long msb = e + qb - 1;
  if (msb > 1023) return sgn * __longlong_as_double(0x7ff0000000000000ll);
  long long lsb = msb - 52 > -1074 ? msb - 52 : -1074;
  long long drop = lsb - e;
  unsigned long long mant;
  if (drop <= 0) mant = q << (-drop);
  else if (drop >= 64) return sgn * 0.0;
  else {
    unsigned long long kept = q >> drop;
    unsigned long long rest = q & ((1ull << drop) - 1);
    unsigned long long half = 1ull << (drop - 1);
    bool up = rest > half || (rest == half && (sticky || (kept & 1)));
    mant = kept + (up ? 1 : 0);
  }
  return sgn * ldexp((double)mant, (int)lsb);
}

struct Sphere { double c[3]; double r2; };

// geometry.py:74-98; returns false on overflow (DegenerateTet)
__device__ __noinline__ bool circumsphere_tet_exact(const double* a, const double* b, const double* c, const double* d, Sphere& s) {
  double xs[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  BI v[12];
  int ex = scaled(xs, 12, v);
  BI u[3], w1[3], w2[3];
  for (int k = 0; k < 3; ++k) { bi_sub(u[k], v[3 + k], v[k]); bi_sub(w1[k], v[6 + k], v[k]); bi_sub(w2[k], v[9 + k], v[k]); }
  BI vw[3], wu[3], uv[3], m1, m2;
  bi_mul(m1, w1[1], w2[2]); bi_mul(m2, w1[2], w2[1]); bi_sub(vw[0], m1, m2);
  bi_mul(m1, w1[2], w2[0]); bi_mul(m2, w1[0], w2[2]); bi_sub(vw[1], m1, m2);
  bi_mul(m1, w1[0], w2[1]); bi_mul(m2, w1[1], w2[0]); bi_sub(vw[2], m1, m2);
  bi_mul(m1, w2[1], u[2]); bi_mul(m2, w2[2], u[1]); bi_sub(wu[0], m1, m2);
  bi_mul(m1, w2[2], u[0]); bi_mul(m2, w2[0], u[2]); bi_sub(wu[1], m1, m2);
  bi_mul(m1, w2[0], u[1]); bi_mul(m2, w2[1], u[0]); bi_sub(wu[2], m1, m2);
  bi_mul(m1, u[1], w1[2]); bi_mul(m2, u[2], w1[1]); bi_sub(uv[0], m1, m2);
  bi_mul(m1, u[2], w1[0]); bi_mul(m2, u[0], w1[2]); bi_sub(uv[1], m1, m2);
  bi_mul(m1, u[0], w1[1]); bi_mul(m2, u[1], w1[0]); bi_sub(uv[2], m1, m2);
  BI den, t1, t2, lu, lv, lw;
  bi_mul(t1, u[0], vw[0]); bi_mul(t2, u[1], vw[1]); bi_add(den, t1, t2); bi_mul(t1, u[2], vw[2]); bi_add(t2, den, t1);
  bi_mulsmall(den, t2, 2);
  bi_mul(t1, u[0], u[0]); bi_mul(t2, u[1], u[1]); bi_add(lu, t1, t2); bi_mul(t1, u[2], u[2]); bi_add(t2, lu, t1); lu = t2;
  bi_mul(t1, w1[0], w1[0]); bi_mul(t2, w1[1], w1[1]); bi_add(lv, t1, t2); bi_mul(t1, w1[2], w1[2]); bi_add(t2, lv, t1); lv = t2;
  bi_mul(t1, w2[0], w2[0]); bi_mul(t2, w2[1], w2[1]); bi_add(lw, t1, t2); bi_mul(t1, w2[2], w2[2]); bi_add(t2, lw, t1); lw = t2;
  BI N[3];
  for (int k = 0; k < 3; ++k) {
    BI x1, x2, x3, s1;
    bi_mul(x1, lu, vw[k]); bi_mul(x2, lv, wu[k]); bi_mul(x3, lw, uv[k]);
    bi_add(s1, x1, x2); bi_add(N[k], s1, x3);
  }
  for (int k = 0; k < 3; ++k) {
    BI num, t;
    bi_mul(t, v[k], den); bi_add(num, t, N[k]);
    s.c[k] = rat_to_double(num, den, ex);
  }
  BI r2n, t, dd;
  bi_mul(r2n, N[0], N[0]); bi_mul(t, N[1], N[1]); bi_add(t1, r2n, t); bi_mul(t, N[2], N[2]); bi_add(r2n, t1, t);
  bi_mul(dd, den, den);
  s.r2 = rat_to_double(r2n, dd, 2 * ex);
  for (int k = 0; k < 3; ++k) if (!isfinite(s.c[k])) return false;
  return isfinite(s.r2);
}

// geometry.py:48-71; returns 0 ok, 1 degenerate (coplanar / overflow)
__device__ __noinline__ int circumsphere_tet(const double* a, const double* b, const double* c, const double* d, Sphere& s) {
  double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
  double v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
  double w0 = d[0] - a[0], w1 = d[1] - a[1], w2 = d[2] - a[2];
  double vw0 = v1 * w2 - v2 * w1, vw1 = v2 * w0 - v0 * w2, vw2 = v0 * w1 - v1 * w0;
  double denom = 2.0 * (u0 * vw0 + u1 * vw1 + u2 * vw2);
  if (denom == 0.0 || !isfinite(denom)) {
    if (orient3d(a, b, c, d) == 0) return 1;
    return circumsphere_tet_exact(a, b, c, d, s) ? 0 : 1;
  }
  double lu = u0 * u0 + u1 * u1 + u2 * u2;
  double lv = v0 * v0 + v1 * v1 + v2 * v2;
  double lw = w0 * w0 + w1 * w1 + w2 * w2;
  double wu0 = w1 * u2 - w2 * u1, wu1 = w2 * u0 - w0 * u2, wu2 = w0 * u1 - w1 * u0;
  double uv0 = u1 * v2 - u2 * v1, uv1 = u2 * v0 - u0 * v2, uv2 = u0 * v1 - u1 * v0;
  double ox = (lu * vw0 + lv * wu0 + lw * uv0) / denom;
  double oy = (lu * vw1 + lv * wu1 + lw * uv1) / denom;
  double oz = (lu * vw2 + lv * wu2 + lw * uv2) / denom;
  s.c[0] = a[0] + ox; s.c[1] = a[1] + oy; s.c[2] = a[2] + oz;
  s.r2 = ox * ox + oy * oy + oz * oz;
  return 0;
}

// geometry.py:101-120; returns false when collinear (DegenerateTri)
__device__ __noinline__ bool circumcircle_tri(const double* a, const double* b, const double* c, Sphere& s) {
  double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
  double v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
  double n0 = u1 * v2 - u2 * v1, n1 = u2 * v0 - u0 * v2, n2 = u0 * v1 - u1 * v0;
  double nn = n0 * n0 + n1 * n1 + n2 * n2;
  if (nn == 0.0) return false;
  double lu = u0 * u0 + u1 * u1 + u2 * u2;
  double lv = v0 * v0 + v1 * v1 + v2 * v2;
  double q0 = lu * v0 - lv * u0, q1 = lu * v1 - lv * u1, q2 = lu * v2 - lv * u2;
  double t0 = q1 * n2 - q2 * n1, t1 = q2 * n0 - q0 * n2, t2 = q0 * n1 - q1 * n0;
  double ox = t0 / (2.0 * nn), oy = t1 / (2.0 * nn), oz = t2 / (2.0 * nn);
  s.c[0] = a[0] + ox; s.c[1] = a[1] + oy; s.c[2] = a[2] + oz;
  s.r2 = ox * ox + oy * oy + oz * oz;
  return true;
}

__device__ __forceinline__ double dist2(const double* a, const double* b) {
  double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

// geometry.py:132-156: p strictly inside the diametral ball of (u,v)
__device__ __forceinline__ bool same_point(const double* a, const double* b) {
  return a[0] == b[0] && a[1] == b[1] && a[2] == b[2];
}
__device__ __noinline__ bool encroaches_segment(const double* u, const double* v, const double* p) {
  double f = 0.0, ssq = 0.0;
  for (int k = 0; k < 3; ++k) {
    double t = 2.0 * p[k] - u[k] - v[k];
    double e = u[k] - v[k];
    f += t * t - e * e;
    ssq += t * t + e * e;
  }
  if (fabs(f) > 1e-12 * ssq) return f < 0.0;
  if (same_point(p, u) || same_point(p, v)) return false;   // an endpoint is on the sphere: f == 0 exactly
  double xs[9] = {p[0], p[1], p[2], u[0], u[1], u[2], v[0], v[1], v[2]};
  BI s[9];
  scaled(xs, 9, s);
  BI total; bi_zero(total);
  for (int k = 0; k < 3; ++k) {
    BI t, e, t2, e2, x, y, tt;
    bi_mulsmall(t2, s[k], 2); bi_sub(x, t2, s[3 + k]); bi_sub(t, x, s[6 + k]);
    bi_sub(e, s[3 + k], s[6 + k]);
    bi_mul(t2, t, t); bi_mul(e2, e, e); bi_sub(y, t2, e2);
    bi_add(tt, total, y); total = tt;
  }
  return total.s < 0;
}

// geometry.py:159-199: sign(|p-o|^2 - r^2) for the equatorial sphere of (a,b,c)
__device__ __noinline__ int equatorial_cmp_exact(const double* a, const double* b, const double* c, const double* p) {
  double xs[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], p[0], p[1], p[2]};
  BI s[12];
  scaled(xs, 12, s);
  BI u[3], v[3], w[3];
  for (int k = 0; k < 3; ++k) { bi_sub(u[k], s[3 + k], s[k]); bi_sub(v[k], s[6 + k], s[k]); bi_sub(w[k], s[9 + k], s[k]); }
  auto dot = [&](BI& out, const BI* x, const BI* y) {
    BI t1, t2, t3;
    bi_mul(t1, x[0], y[0]); bi_mul(t2, x[1], y[1]); bi_add(t3, t1, t2); bi_mul(t1, x[2], y[2]); bi_add(out, t3, t1);
  };
  BI uu, vv, uv, ww, uw, vw, det, t1, t2, c1, c2, val, tmp;
  dot(uu, u, u); dot(vv, v, v); dot(uv, u, v); dot(ww, w, w); dot(uw, u, w); dot(vw, v, w);
  bi_mul(t1, uu, vv); bi_mul(t2, uv, uv); bi_sub(det, t1, t2);
  if (det.s == 0) { raise_err(GQ_ERR_DEGEN); return 1; }
  // c1 = uu*vv - uv*vv ; c2 = vv*uu - uv*uu
  bi_mul(t2, uv, vv); bi_sub(c1, t1, t2);
  bi_mul(t2, uv, uu); bi_sub(c2, t1, t2);
  bi_mul(val, det, ww);
  bi_mul(t1, c1, uw); bi_sub(tmp, val, t1);
  bi_mul(t1, c2, vw); bi_sub(val, tmp, t1);
  return val.s;
}
__device__ __noinline__ int equatorial_cmp(const double* a, const double* b, const double* c, const double* p) {
  Sphere sph;
  if (!circumcircle_tri(a, b, c, sph)) { raise_err(GQ_ERR_DEGEN); return 1; }
  double f = dist2(p, sph.c) - sph.r2;
  double scale = dist2(p, sph.c) + sph.r2;
  if (fabs(f) > 1e-9 * scale) return f > 0 ? 1 : -1;
  // a vertex of the triangle lies exactly on its equatorial sphere
  if (same_point(p, a) || same_point(p, b) || same_point(p, c)) return 0;
  return equatorial_cmp_exact(a, b, c, p);
}
// The same comparison for the in-plane Delaunay test of oblique polygons:
// sliver triangles (split points along one subsegment) can make the float
// circumcircle degenerate; the exact evaluation decides them.
__device__ __noinline__ int equatorial_cmp_robust(const double* a, const double* b, const double* c, const double* p) {
  if (same_point(p, a) || same_point(p, b) || same_point(p, c)) return 0;
  Sphere sph;
  if (circumcircle_tri(a, b, c, sph)) {
    double f = dist2(p, sph.c) - sph.r2;
    double scale = dist2(p, sph.c) + sph.r2;
    if (isfinite(f) && fabs(f) > 1e-9 * scale) return f > 0 ? 1 : -1;
  }
  return equatorial_cmp_exact(a, b, c, p);
}
__device__ inline bool encroaches_face(const double* a, const double* b, const double* c, const double* p) {
  return equatorial_cmp(a, b, c, p) < 0;
}

// facets.py:99-104: p on the line of (a,b) strictly between a and b (exact)
__device__ __noinline__ bool between2d_exact(const double* a, const double* b, const double* p) {
  double xs[6] = {p[0], p[1], a[0], a[1], b[0], b[1]};
  BI v[6];
  scaled(xs, 6, v);
  BI x0, x1, y0, y1, t1, t2, d0, dl;
  bi_sub(x0, v[0], v[2]); bi_sub(y0, v[4], v[2]); bi_mul(t1, x0, y0);
  bi_sub(x1, v[1], v[3]); bi_sub(y1, v[5], v[3]); bi_mul(t2, x1, y1);
  bi_add(d0, t1, t2);
  bi_mul(t1, y0, y0); bi_mul(t2, y1, y1); bi_add(dl, t1, t2);
  if (d0.s <= 0) return false;
  BI diff; bi_sub(diff, d0, dl);
  return diff.s < 0;
}

}  // namespace gq
