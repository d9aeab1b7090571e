// gq_grid.cuh -- constraint-ball grid, the device ConstraintIndex (refine.py:107-253, 314-335).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

// ---------------------------------------------------------------------------
// constraint-ball grid: the reference's ConstraintIndex (refine.py:107-253)
// on the device.  Every live subsegment / subface ball is listed in the cells
// its bounding box overlaps, on the finest level of a multi-level grid where
// that is at most 3 cells per axis (CSR lists, rebuilt from the live records).
// Queries only enumerate candidates; decisions are the exact open-ball
// predicates.
struct CGrid {
  double lo[3], inv[3];
  int G;              // level-0 cells per axis
  int L;              // levels: level l has ceil(G / 2^l) cells per axis, the last has 1
  int off[16];        // first cell of each level in start[]
  int ncell;          // total cells over all levels
  int* start;         // ncell + 1: CSR offsets of the cell lists (live balls only)
  int* codes;         // 2*rec + kind
  int* cnt;           // ncell + 1 counters / fill cursors
  int node_cap;
  int* nbig;          // [1] = CSR overflow flag
};
__device__ __host__ __forceinline__ int cg_gl(int G, int l) { return (G + (1 << l) - 1) >> l; }
__device__ __forceinline__ int cg_ci(const CGrid& g, double x, int k) {
  double f = (x - g.lo[k]) * g.inv[k];
  if (!(f >= 0.0)) return 0;
  if (f >= (double)g.G) return g.G - 1;
  return (int)f;
}
__device__ inline bool cons_ball(const Dev& D, int kind, int r, double* c, double& r2) {
  if (kind == 0) {
    int2 e = D.sg_uv[r];
    const double *pu = PT(D, e.x), *pv = PT(D, e.y);
    for (int k = 0; k < 3; ++k) c[k] = (pu[k] + pv[k]) / 2.0;
    r2 = (pu[0] - c[0]) * (pu[0] - c[0]) + (pu[1] - c[1]) * (pu[1] - c[1]) + (pu[2] - c[2]) * (pu[2] - c[2]);
    return true;
  }
  int4 f = D.sf_v[r];
  Sphere s;
  if (!circumcircle_tri(PT(D, f.x), PT(D, f.y), PT(D, f.z), s)) return false;
  c[0] = s.c[0]; c[1] = s.c[1]; c[2] = s.c[2]; r2 = s.r2;
  return true;
}
// The grid is rebuilt from the live records whenever it is queried after a
// change (count -> scan -> fill): cell lists are contiguous and hold no dead
// records.  Levels halve the resolution; a ball is stored at the finest level
// where it spans at most 3 cells per axis, so a query reads one short run per
// level and there is no "big ball" list scanned by everyone.
// pass 0 counts, pass 1 fills.
__global__ void k_grid_build(const __grid_constant__ Dev D, CGrid g, int nseg, int nface, int pass) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nseg + nface; x += gridDim.x * blockDim.x) {
    int kind = x < nseg ? 0 : 1, r = x < nseg ? x : x - nseg;
    unsigned int fl = kind == 0 ? D.sg_fl[r] : D.sf_fl[r];
    if (!(fl & RF_LIVE)) continue;
    double c[3], r2;
    if (!cons_ball(D, kind, r, c, r2)) continue;
    double rr = sqrt(r2) * (1.0 + 1e-9) + 1e-300;
    int i0 = cg_ci(g, c[0] - rr, 0), i1 = cg_ci(g, c[0] + rr, 0);
    int j0 = cg_ci(g, c[1] - rr, 1), j1 = cg_ci(g, c[1] + rr, 1);
    int k0 = cg_ci(g, c[2] - rr, 2), k1 = cg_ci(g, c[2] + rr, 2);
    int l = 0;
    while (l < g.L - 1 && ((i1 >> l) - (i0 >> l) > 2 || (j1 >> l) - (j0 >> l) > 2 || (k1 >> l) - (k0 >> l) > 2)) ++l;
    const int Gl = cg_gl(g.G, l), base = g.off[l];
    int code = 2 * r + kind;
    for (int i = i0 >> l; i <= i1 >> l; ++i) for (int j = j0 >> l; j <= j1 >> l; ++j) for (int k = k0 >> l; k <= k1 >> l; ++k) {
      int cell = base + (i * Gl + j) * Gl + k;
      if (pass == 0) { atomicAdd(g.cnt + cell, 1); continue; }
      int pos = g.start[cell] + atomicAdd(g.cnt + cell, 1);
      if (pos < g.node_cap) g.codes[pos] = code; else if (atomicExch(g.nbig + 1, 1) == 0) raise_err(GQ_ERR_CAP);
    }
  }
}
// visit every live constraint whose open ball strictly contains p
template <class F>
__device__ inline void grid_encroached(const Dev& D, const CGrid& g, const double* p, int kinds, F f) {
  const int ci = cg_ci(g, p[0], 0), cj = cg_ci(g, p[1], 1), ck = cg_ci(g, p[2], 2);
  auto test = [&](int code) {
    int kind = code & 1, r = code >> 1;
    if (!((kinds >> kind) & 1)) return;
    if (kind == 0) {
      if (!(D.sg_fl[r] & RF_LIVE)) return;
      int2 e = D.sg_uv[r];
      if (encroaches_segment(PT(D, e.x), PT(D, e.y), p)) f(0, r);
    } else {
      if (!(D.sf_fl[r] & RF_LIVE)) return;
      int4 q = D.sf_v[r];
      if (encroaches_face(PT(D, q.x), PT(D, q.y), PT(D, q.z), p)) f(1, r);
    }
  };
  for (int l = 0; l < g.L; ++l) {
    const int Gl = cg_gl(g.G, l);
    const int cell = g.off[l] + ((ci >> l) * Gl + (cj >> l)) * Gl + (ck >> l);
    const int e = g.start[cell + 1];
    for (int k = g.start[cell]; k < e; ++k) test(g.codes[k]);
  }
}
// A query's cell lists can run to hundreds of balls (coarse levels, few and
// large constraints early on): the warp versions below scan them 32 at a time.
__device__ inline int grid_hit(const Dev& D, int code, const double* p, int kinds) {   // kind hit, or -1
  int kind = code & 1, r = code >> 1;
  if (!((kinds >> kind) & 1)) return -1;
  if (kind == 0) {
    if (!(D.sg_fl[r] & RF_LIVE)) return -1;
    int2 e = D.sg_uv[r];
    return encroaches_segment(PT(D, e.x), PT(D, e.y), p) ? 0 : -1;
  }
  if (!(D.sf_fl[r] & RF_LIVE)) return -1;
  int4 q = D.sf_v[r];
  return encroaches_face(PT(D, q.x), PT(D, q.y), PT(D, q.z), p) ? 1 : -1;
}
// warp-uniform p; f(kind, rec, hit) is called by every lane once per chunk of
// 32 list entries (hit false on lanes without one), so callers can ballot
template <class F>
__device__ inline void grid_encroached_warp(const Dev& D, const CGrid& g, const double* p, int kinds, F f) {
  const int lane = threadIdx.x & 31;
  const int ci = cg_ci(g, p[0], 0), cj = cg_ci(g, p[1], 1), ck = cg_ci(g, p[2], 2);
  for (int l = 0; l < g.L; ++l) {
    const int Gl = cg_gl(g.G, l);
    const int cell = g.off[l] + ((ci >> l) * Gl + (cj >> l)) * Gl + (ck >> l);
    const int s = g.start[cell], e = g.start[cell + 1];
    for (int b = s; b < e; b += 32) {
      int k = b + lane, kind = -1, r = -1;
      if (k < e) { int code = g.codes[k]; r = code >> 1; kind = grid_hit(D, code, p, kinds); }
      f(kind, r);
    }
  }
}
#define GRID_WARP0 ((int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5))
#define GRID_NWARP ((int)((gridDim.x * blockDim.x) >> 5))
__global__ void k_grid_newverts_w(const __grid_constant__ Dev D, CGrid g, int v0, int v1) {
  for (int v = v0 + GRID_WARP0; v < v1; v += GRID_NWARP)
    grid_encroached_warp(D, g, PT(D, v), 3, [&](int kind, int r) {
      if (kind < 0) return;
      unsigned int* fl = kind == 0 ? D.sg_fl + r : D.sf_fl + r;
      if (!(*fl & RF_SKIP)) atomicOr(fl, RF_ENC);
    });
}
__global__ void k_grid_cands_w(const __grid_constant__ Dev D, CGrid g, const __grid_constant__ Cand C, int n0, int n1) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int c = n0 + GRID_WARP0; c < n1; c += GRID_NWARP) {
    int kind = C.kind[c];
    if (kind == K_SEG || C.status[c] == CS_DROP) {
      if (lane == 0) { C.nrseg[c] = 0; C.nrface[c] = 0; }
      continue;
    }
    int ns = 0, nf = 0;
    int* rs = C.rseg + (size_t)c * CRD;
    int* rf = C.rface + (size_t)c * CRD;
    grid_encroached_warp(D, g, C.p + 3 * (size_t)c, kind == K_TET ? 3 : 1, [&](int k, int r) {
      bool hs = k == 0 && !(D.sg_fl[r] & RF_SKIP), hf = k == 1 && !(D.sf_fl[r] & RF_SKIP);
      unsigned ms = __ballot_sync(0xffffffffu, hs), mf = __ballot_sync(0xffffffffu, hf);
      if (hs) { int q = ns + __popc(ms & lt); if (q < CRD) rs[q] = r; else raise_err(GQ_ERR_CAP); }
      if (hf) { int q = nf + __popc(mf & lt); if (q < CRD) rf[q] = r; else raise_err(GQ_ERR_CAP); }
      ns += __popc(ms); nf += __popc(mf);
    });
    if (lane == 0) { C.nrseg[c] = ns < CRD ? ns : CRD; C.nrface[c] = nf < CRD ? nf : CRD; }
  }
}
// post_round part 1 (refine.py:818-828): new vertices against all balls
__global__ void k_grid_newverts(const __grid_constant__ Dev D, CGrid g, int v0, int v1) {
  for (int v = v0 + blockIdx.x * blockDim.x + threadIdx.x; v < v1; v += gridDim.x * blockDim.x) {
    grid_encroached(D, g, PT(D, v), 3, [&](int kind, int r) {
      unsigned int* fl = kind == 0 ? D.sg_fl + r : D.sf_fl + r;
      if (!(*fl & RF_SKIP)) atomicOr(fl, RF_ENC);
    });
  }
}
// redirect hits of candidate points (refine.py:603-613, 636-654)
__global__ void k_grid_cands(const __grid_constant__ Dev D, CGrid g, const __grid_constant__ Cand C, int n0, int n1) {
  for (int c = n0 + blockIdx.x * blockDim.x + threadIdx.x; c < n1; c += gridDim.x * blockDim.x) {
    int kind = C.kind[c];
    C.nrseg[c] = 0; C.nrface[c] = 0;
    if (kind == K_SEG || C.status[c] == CS_DROP) continue;
    int ns = 0, nf = 0;
    int* rs = C.rseg + (size_t)c * CRD;
    int* rf = C.rface + (size_t)c * CRD;
    grid_encroached(D, g, C.p + 3 * (size_t)c, kind == K_TET ? 3 : 1, [&](int k, int r) {
      if (k == 0) { if (D.sg_fl[r] & RF_SKIP) return; if (ns < CRD) rs[ns++] = r; else raise_err(GQ_ERR_CAP); }
      else { if (D.sf_fl[r] & RF_SKIP) return; if (nf < CRD) rf[nf++] = r; else raise_err(GQ_ERR_CAP); }
    });
    C.nrseg[c] = ns; C.nrface[c] = nf;
  }
}

