// gq_setup.cuh -- device certification of PLC validity.
//
// The reference validates a PLC in exact rational arithmetic, one feature pair
// at a time (plc.py:267-383): hours for C4's 306k segments and 204k triangles.
// The structural checks (indices, duplicates, degenerate triangles, polygon
// edges) are cheap vectorised host work; what remains is every pair of
// features whose boxes overlap:
//   * candidate pairs from a uniform grid over the feature boxes (features
//     spanning more than 3 cells per axis are tested against everything),
//     each pair reported once, in the first cell both boxes share;
//   * segment / segment and segment / triangle conflicts decided with the
//     exact device predicates, mirroring the vectorised certifier of
//     setup_fast.py: a pair is either cleared, a certain conflict, or handed
//     back to the host's exact pair test (coplanar / collinear degeneracies).
// Polygon / polygon pairs are not tested, as in the reference (an interior
// crossing always crosses a boundary segment).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

struct CertIn {
  const double* P;      // points
  const int* seg;       // m x 2
  const int* tri;       // f x 3
  int m, f;
  double lo[3], inv;    // grid origin, 1 / cell size
  int G[3];             // cells per axis
};
__device__ inline void cert_box(const CertIn& I, int k, double* lo, double* hi) {
  int nv = k < I.m ? 2 : 3;
  const int* id = k < I.m ? I.seg + 2 * (size_t)k : I.tri + 3 * (size_t)(k - I.m);
  for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
  for (int j = 0; j < nv; ++j) {
    const double* p = I.P + 3 * (size_t)id[j];
    for (int a = 0; a < 3; ++a) { lo[a] = fmin(lo[a], p[a]); hi[a] = fmax(hi[a], p[a]); }
  }
}
__device__ inline void cert_cells(const CertIn& I, const double* lo, const double* hi, int* i0, int* i1) {
  for (int a = 0; a < 3; ++a) {
    double f0 = (lo[a] - I.lo[a]) * I.inv, f1 = (hi[a] - I.lo[a]) * I.inv;
    i0[a] = min(max((int)floor(f0), 0), I.G[a] - 1);
    i1[a] = min(max((int)floor(f1), 0), I.G[a] - 1);
  }
}
__device__ inline bool cert_big(const int* i0, const int* i1) { return i1[0] - i0[0] >= 3 || i1[1] - i0[1] >= 3 || i1[2] - i0[2] >= 3; }
__device__ inline int cert_cell(const CertIn& I, int x, int y, int z) { return (x * I.G[1] + y) * I.G[2] + z; }

__global__ void k_cert_extent(CertIn I, double* ext) {
  int n = I.m + I.f;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double lo[3], hi[3];
    cert_box(I, k, lo, hi);
    ext[k] = fmax(hi[0] - lo[0], fmax(hi[1] - lo[1], hi[2] - lo[2]));
  }
}
// pass 0: count per cell (+ big list), pass 1: fill
__global__ void k_cert_bin(CertIn I, int* cnt, const int* start, int* fillpos, int* lists, int* big, int* nbig, int pass) {
  int n = I.m + I.f;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double lo[3], hi[3];
    int i0[3], i1[3];
    cert_box(I, k, lo, hi);
    cert_cells(I, lo, hi, i0, i1);
    if (cert_big(i0, i1)) { if (pass == 0) big[atomicAdd(nbig, 1)] = k; continue; }
    for (int x = i0[0]; x <= i1[0]; ++x)
      for (int y = i0[1]; y <= i1[1]; ++y)
        for (int z = i0[2]; z <= i1[2]; ++z) {
          int cidx = cert_cell(I, x, y, z);
          if (pass == 0) atomicAdd(cnt + cidx, 1);
          else lists[start[cidx] + atomicAdd(fillpos + cidx, 1)] = k;
        }
  }
}

// 0 clear, 1 certain conflict, 2 undecided (host exact test).  u < v.
__device__ int cert_pair(const CertIn& I, int u, int v) {
  if (u >= I.m) return 0;                                  // polygon / polygon: not tested (plc.py:380-381)
  const double* P = I.P;
  int a = I.seg[2 * u], b = I.seg[2 * u + 1];
  const double *pa = P + 3 * (size_t)a, *pb = P + 3 * (size_t)b;
  if (v < I.m) {                                           // segment / segment
    int c = I.seg[2 * v], d = I.seg[2 * v + 1];
    bool share = a == c || a == d || b == c || b == d;
    if (!share) return orient3d(pa, pb, P + 3 * (size_t)c, P + 3 * (size_t)d) != 0 ? 0 : 2;
    int other = (c == a || c == b) ? d : c;
    const double* po = P + 3 * (size_t)other;
    // one shared endpoint: a conflict needs the three points collinear
    double x0[2] = {pa[1], pa[2]}, x1[2] = {pb[1], pb[2]}, x2[2] = {po[1], po[2]};
    double y0[2] = {pa[0], pa[2]}, y1[2] = {pb[0], pb[2]}, y2[2] = {po[0], po[2]};
    double z0[2] = {pa[0], pa[1]}, z1[2] = {pb[0], pb[1]}, z2[2] = {po[0], po[1]};
    bool collinear = orient2d(x0, x1, x2) == 0 && orient2d(y0, y1, y2) == 0 && orient2d(z0, z1, z2) == 0;
    return collinear ? 2 : 0;
  }
  const int* T = I.tri + 3 * (size_t)(v - I.m);            // segment / triangle
  bool in_i = T[0] == a || T[1] == a || T[2] == a;
  bool in_j = T[0] == b || T[1] == b || T[2] == b;
  if (in_i && in_j) return 0;                              // a side of the triangle
  const double *p0 = P + 3 * (size_t)T[0], *p1 = P + 3 * (size_t)T[1], *p2 = P + 3 * (size_t)T[2];
  int sa = in_i ? 0 : orient3d(p0, p1, p2, pa);
  int sb = in_j ? 0 : orient3d(p0, p1, p2, pb);
  if (sa * sb > 0) return 0;                               // both strictly on one side
  if ((sa == 0 && in_i && sb != 0) || (sb == 0 && in_j && sa != 0)) return 0;   // touches at its own vertex
  if (sa * sb < 0 && !in_i && !in_j) {                     // proper plane crossing
    const double* q[3] = {p0, p1, p2};
    int o[3];
    for (int k = 0; k < 3; ++k) o[k] = orient3d(pa, pb, q[k], q[(k + 1) % 3]);
    bool pos = o[0] > 0 || o[1] > 0 || o[2] > 0, neg = o[0] < 0 || o[1] < 0 || o[2] < 0;
    if (pos && neg) return 0;                              // the line misses the closed triangle
    if ((o[0] > 0 && o[1] > 0 && o[2] > 0) || (o[0] < 0 && o[1] < 0 && o[2] < 0)) return 1;   // interior hit
    return 2;
  }
  return 2;
}
struct CertOut { int* flag; int* pairs; int cap; int* npairs; };
__device__ inline void cert_report(const CertOut& O, int r, int u, int v) {
  if (r == 1) { atomicOr(O.flag, 1); return; }
  if (r == 2) {
    int k = atomicAdd(O.npairs, 1);
    if (k < O.cap) { O.pairs[2 * k] = u; O.pairs[2 * k + 1] = v; } else atomicOr(O.flag, 2);
  }
}
__device__ inline bool boxes_overlap(const double* alo, const double* ahi, const double* blo, const double* bhi) {
  return alo[0] <= bhi[0] && blo[0] <= ahi[0] && alo[1] <= bhi[1] && blo[1] <= ahi[1] && alo[2] <= bhi[2] && blo[2] <= ahi[2];
}
// small features: pairs met in a shared cell, kept in the first cell both boxes cover
__global__ void k_cert_pairs(CertIn I, const int* start, const int* lists, CertOut O) {
  int n = I.m + I.f;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    double lo[3], hi[3];
    int i0[3], i1[3];
    cert_box(I, u, lo, hi);
    cert_cells(I, lo, hi, i0, i1);
    if (cert_big(i0, i1)) continue;
    for (int x = i0[0]; x <= i1[0]; ++x)
      for (int y = i0[1]; y <= i1[1]; ++y)
        for (int z = i0[2]; z <= i1[2]; ++z) {
          int cidx = cert_cell(I, x, y, z);
          for (int q = start[cidx]; q < start[cidx + 1]; ++q) {
            int v = lists[q];
            if (v <= u) continue;
            double vlo[3], vhi[3];
            int j0[3], j1[3];
            cert_box(I, v, vlo, vhi);
            cert_cells(I, vlo, vhi, j0, j1);
            if (max(i0[0], j0[0]) != x || max(i0[1], j0[1]) != y || max(i0[2], j0[2]) != z) continue;
            if (!boxes_overlap(lo, hi, vlo, vhi)) continue;
            cert_report(O, cert_pair(I, u, v), u, v);
          }
        }
  }
}
// big features against every other feature (pairs of two big ones once)
__global__ void k_cert_big(CertIn I, const int* big, int nbig, CertOut O) {
  int n = I.m + I.f;
  long long tot = (long long)nbig * n;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < tot; w += (long long)gridDim.x * blockDim.x) {
    int b = big[w / n], v = (int)(w % n);
    if (v == b) continue;
    double lo[3], hi[3], vlo[3], vhi[3];
    int i0[3], i1[3];
    cert_box(I, v, vlo, vhi);
    cert_cells(I, vlo, vhi, i0, i1);
    if (cert_big(i0, i1) && v < b) continue;               // the other big one reports it
    cert_box(I, b, lo, hi);
    if (!boxes_overlap(lo, hi, vlo, vhi)) continue;
    int u0 = min(b, v), v0 = max(b, v);
    cert_report(O, cert_pair(I, u0, v0), u0, v0);
  }
}
