// gq_warp.cuh -- warp-cooperative Delaunay region (the common case).
//
// One warp computes one candidate's region with the decisions of
// region_compute() (mesh.py:450-521 / _kernels.py:392-635): the 32 lanes
// test the frontier's neighbours in parallel (FP-filtered insphere /
// orient3d with the exact fallback), the grown set is a per-warp
// shared-memory hash, peel / component are warp passes, and the finished
// cavity is sorted (warp bitonic) and its boundary faces emitted through a
// warp scan in the reference order.  Cavities larger than WR_MAXT tets
// report RS_OVERFLOW and go to the block kernel (gq_block.cuh).
#pragma once
#include "gq_dev.cuh"

namespace gq {

#ifdef GQ_DCHECK
#define DCHK(cond, ...) do { if (!(cond)) { printf("DCHECK %s:%d " #cond "\n", __FILE__, __LINE__); raise_err(GQ_ERR_CAP); } } while (0)
#else
#define DCHK(cond, ...) do {} while (0)
#endif

__device__ int g_wstop;
__device__ volatile int* g_wdbg;      // pinned host mirror: [warp][2] = candidate, checkpoint
#ifdef GQ_DCHECK
#define WMARK(k) do { if (g_wdbg) { int gt_ = blockIdx.x * blockDim.x + threadIdx.x; g_wdbg[40000 + gt_] = (k) * 1000 + __LINE__ % 1000; } } while (0)
#else
#define WMARK(k) do {} while (0)
#endif
#define WSTOP(k) do { if (g_wstop == (k)) return RS_CNSS; } while (0)
#ifndef CC_DBG
#define CC_DBG 96
#endif
#ifndef WR_WARPS
#define WR_WARPS 4          // warps per block (C2: 4 measured 538 ms vs 543 ms for 8, same occupancy at 233 registers)
#endif

// Two instantiations: a small tier (128 tets, 6.5 KB per warp) that runs at
// 16 warps / SM for the common cavities, and a large tier (512 tets, 25 KB per
// warp) for the few percent that overflow the small one.
template <int MAXT, int HASH>
struct WarpSharedT {
  int hkey[HASH];
  short hval[HASH];          // cavity index (< MAXT) or -2 (tested, outside)
  int cav[MAXT];
  int f0[MAXT];
  int f1[MAXT];
  int comp[MAXT];
  unsigned char in[MAXT];
  int n, nf, cnt, flag, memb, seed, ghost, seedk;
  unsigned long long mind;
  int seeds[32];
  int nseeds;
};

template <int HASH>
__device__ __forceinline__ unsigned int wh(int k) { return ((unsigned int)k * 2654435761u) & (HASH - 1); }
template <class WS>
__device__ inline int wh_claim(WS& W, int k) {
  constexpr int HASH = sizeof(W.hkey) / sizeof(int);
  unsigned int i = wh<HASH>(k);
  for (int p = 0; p < HASH; ++p) {
    int cur = W.hkey[i];
    if (cur == k) return -1;
    if (cur == INT_MIN) {
      int old = atomicCAS(&W.hkey[i], INT_MIN, k);
      if (old == INT_MIN) return (int)i;
      if (old == k) return -1;
    }
    i = (i + 1) & (HASH - 1);
  }
  return -2;
}
template <class WS>
__device__ inline int wh_find(const WS& W, int k) {
  constexpr int HASH = sizeof(W.hkey) / sizeof(int);
  unsigned int i = wh<HASH>(k);
  for (int p = 0; p < HASH; ++p) {
    int cur = W.hkey[i];
    if (cur == k) return W.hval[i];
    if (cur == INT_MIN) return -1;
    i = (i + 1) & (HASH - 1);
  }
  return -1;
}

// bf_open_part for a warp with the boundary faces' vertex triples staged in
// shared memory first (the cavity hash is free at this point and is cleared
// again right after): the pairing count reads shared memory instead of
// gathering every face's vertices from the mesh nbf times.  Same answer.
__device__ inline bool bf_open_warp(const Dev& D, const int* bf, int nbf, int* sh, int shcap, int lane) {
  if (3 * nbf > shcap) return __any_sync(0xffffffffu, bf_open_part(D, bf, nbf, lane, 32));
  for (int k = lane; k < nbf; k += 32) {
    int f[3]; face_verts(D.tv[bf[k] >> 2], bf[k] & 3, f);
    sh[3 * k] = f[0]; sh[3 * k + 1] = f[1]; sh[3 * k + 2] = f[2];
  }
  __syncwarp();
  bool open = false;
  for (int k = lane; k < nbf && !open; k += 32) {
    for (int e = 0; e < 3 && !open; ++e) {
      const int x = sh[3 * k + e], y = sh[3 * k + (e + 1) % 3];
      int cnt = 0;
      for (int j = 0; j < nbf && cnt <= 2; ++j) {
        const int a = sh[3 * j], b = sh[3 * j + 1], c = sh[3 * j + 2];
        cnt += (a == x || b == x || c == x) && (a == y || b == y || c == y);
      }
      open = cnt != 2;
    }
  }
  const bool r = __any_sync(0xffffffffu, open);
  __syncwarp();
  return r;
}

// All 32 lanes of the warp call this with the same arguments.  S is the
// warp's global scratch (lane 0 only: walks and the constraint pass).
template <int MAXT, int HASH>
__device__ inline int region_warp(const Dev& D, const double* p, const int* seeds, int nseeds, const Allow& A,
                                  WarpSharedT<MAXT, HASH>& W, Scratch& S, RegionOut& O, bool walk_on_miss = true,
                                  unsigned excl = 0u, bool may_retry = false, bool check_ghost = true) {
  constexpr int WR_MAXT = MAXT, WR_HASH = HASH;
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  for (int i = lane; i < WR_HASH; i += 32) W.hkey[i] = INT_MIN;
  __syncwarp();
  // seed: first listed alive tet whose region contains p (tests in parallel)
  int nc = nseeds < 32 ? nseeds : 32;
  int t0 = lane < nc ? seeds[lane] : -1;
  DCHK(t0 < D.tcap);
  bool ok = t0 >= 0 && !((excl >> lane) & 1u) && D.alive[t0] && in_region(D, t0, p, A);
  unsigned bal = __ballot_sync(FULL, ok);
  int seed = bal ? __shfl_sync(FULL, t0, __ffs(bal) - 1) : -1;
  if (lane == 0) W.seedk = bal ? __ffs(bal) - 1 : -1;   // which listed seed (region_warp_retry)
  if (seed < 0 && excl) return RS_CNSS;                 // a retry with no further seed
  if (seed < 0) {
    WMARK(50);
    if (!walk_on_miss) return RS_CNSS;
    if (lane == 0) {
      int t = walk(D, p, nc > 0 ? seeds[0] : -1);
      W.seed = (t >= 0 && D.alive[t] && in_region(D, t, p, A)) ? t : -1;
    }
    __syncwarp();
    seed = W.seed;
    WMARK(50);
    if (seed < 0) {
      if (lane == 0) {
        unsigned k = atomicAdd(&D.ctr->fail[0], 1u);
#ifdef GQ_DEBUG2D
        if (k < 40) {
          int t0s = seeds[0];
          int4 q = D.tv[t0s];
          printf("[noseed] k %u nseeds %d p %.17g %.17g %.17g seed0 %d alive %d tv %d %d %d %d walk %d insph %d\n", k, nseeds,
                 p[0], p[1], p[2], t0s, (int)D.alive[t0s], q.x, q.y, q.z, q.w, W.seed,
                 q.w == GHOST ? -9 : insphere(PT(D, q.x), PT(D, q.y), PT(D, q.z), PT(D, q.w), p));
          for (int j = 0; j < 4; ++j) {
            int v = tvk(q, j);
            if (v == GHOST) continue;
            const double* a = PT(D, v);
            double d2 = (a[0] - p[0]) * (a[0] - p[0]) + (a[1] - p[1]) * (a[1] - p[1]) + (a[2] - p[2]) * (a[2] - p[2]);
            if (d2 == 0.0) printf("[noseed]   k %u coincides with vertex %d origin %d vsid %d\n", k, v, (int)D.vorigin[v], D.vsid[v]);
          }
        }
#else
        (void)k;
#endif
      }
      return RS_CNSS;
    }
  }
  O.seed = seed;
  WSTOP(1);
  WMARK(11);
  if (lane == 0) {
    int s = wh_claim(W, seed);       // the table is empty: always inserts
    if (s >= 0) W.hval[s] = 0;
    W.cav[0] = seed; W.n = 1; W.f0[0] = seed; W.flag = 0; W.memb = INT_MAX; W.ghost = D.tv[seed].w == GHOST;
  }
  __syncwarp();
  // ---- grow
  int* cur = W.f0; int* nxt = W.f1;
  int ncur = 1;
  while (ncur > 0) {
    if (lane == 0) W.nf = 0;
    __syncwarp();
    for (int j = lane; j < 4 * ncur; j += 32) {
      DCHK((j >> 2) < WR_MAXT);
      int t = cur[j >> 2], i = j & 3;
      DCHK(t >= 0 && t < D.tcap);
      int u = tnk(D, t, i) >> 2;
      DCHK(u < D.tcap);
      if (u < 0 || !D.alive[u]) continue;
      if (blocked(D, A, t, i)) continue;
      int slot = wh_claim(W, u);
      if (slot == -1) continue;
      if (slot == -2) { W.flag = 1; continue; }
      if (in_region(D, u, p, A)) {
        int idx = atomicAdd(&W.n, 1);
        if (idx >= WR_MAXT) { W.flag = 1; W.hval[slot] = -2; continue; }
        W.cav[idx] = u;
        W.hval[slot] = idx;
        nxt[atomicAdd(&W.nf, 1)] = u;
        if (D.tv[u].w == GHOST) W.ghost = 1;   // only a ghost tet puts ghost faces on the boundary
      } else {
        W.hval[slot] = -2;
      }
    }
    __syncwarp();
    WMARK(50);
    if (W.flag) return RS_OVERFLOW;
    ncur = W.nf;
    int* tmp = cur; cur = nxt; nxt = tmp;
    __syncwarp();
  }
  const int n = W.n;
  WSTOP(2);
  WMARK(12);
  // ---- peel / seed component (confluent fixpoint)
  for (int k = lane; k < n; k += 32) W.in[k] = 1;
  __syncwarp();
  while (true) {
    while (true) {
      WMARK(20);
      bool changed = false;
      for (int k = lane; k < n; k += 32) {
        if (!W.in[k]) continue;
        int t = W.cav[k];
        DCHK(t >= 0 && t < D.tcap);
        int4 q = D.tv[t];
        for (int i = 0; i < 4; ++i) {
          int u = tnk(D, t, i) >> 2;
          bool blk = blocked(D, A, t, i);
          int ku = wh_find(W, u);
          DCHK(ku < WR_MAXT);
          bool uin = ku >= 0 && W.in[ku];
          if (uin && !blk) continue;
          int f[3]; face_verts(q, i, f);
          if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) continue;
          if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) >= 0) { W.in[k] = 0; changed = true; break; }
        }
      }
      __syncwarp();
      if (!__any_sync(FULL, changed)) break;
    }
    WMARK(50);
    const bool shrunk = !W.in[0];
    __syncwarp();
    if (shrunk) {   // seed shrunk away
      if (may_retry && W.seedk >= 0 && D.poly_obl_hull) return RS_SHRUNK;   // the caller may retry
      if (lane == 0) {
        unsigned k = atomicAdd(&D.ctr->fail[1], 1u);
#ifdef GQ_DEBUG2D
        if (k < 40) {
          int4 q = D.tv[seed];
          printf("[peeled] k %u n %d p %.17g %.17g %.17g seed %d tv %d %d %d %d nseeds %d\n", k, n, p[0], p[1], p[2], seed,
                 q.x, q.y, q.z, q.w, nseeds);
        }
#else
        (void)k;
#endif
      }
      return RS_CNSS;
    }
    for (int k = lane; k < n; k += 32) W.comp[k] = 0;
    __syncwarp();
    if (lane == 0) { W.comp[0] = 1; W.f0[0] = 0; W.cnt = 1; }
    __syncwarp();
    WMARK(21);
    int* fa = W.f0; int* fb = W.f1;
    int nfa = 1;
    while (nfa > 0) {
      if (lane == 0) W.nf = 0;
      __syncwarp();
      for (int j = lane; j < 4 * nfa; j += 32) {
        int k = fa[j >> 2], i = j & 3;
        int t = W.cav[k];
        int u = tnk(D, t, i) >> 2;
        int ku = wh_find(W, u);
        if (ku < 0 || !W.in[ku]) continue;
        if (blocked(D, A, t, i)) continue;
        if (atomicCAS(&W.comp[ku], 0, 1) != 0) continue;
        atomicAdd(&W.cnt, 1);
        fb[atomicAdd(&W.nf, 1)] = ku;
      }
      __syncwarp();
      nfa = W.nf;
      int* tmp = fa; fa = fb; fb = tmp;
      __syncwarp();
    }
    int live = 0;
    for (int k = lane; k < n; k += 32) live += W.in[k];
    for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(FULL, live, o);
    const bool done = W.cnt == live;
    __syncwarp();                 // every lane has read W.cnt before anyone moves on
    if (done) break;
    for (int k = lane; k < n; k += 32) W.in[k] = (unsigned char)W.comp[k];
    __syncwarp();
  }
  WSTOP(3);
  WMARK(13);
  // ---- finish: members, sorted by tet id (warp bitonic over 128 slots)
  if (lane == 0) W.cnt = 0;
  __syncwarp();
  for (int k = lane; k < n; k += 32) if (W.in[k]) W.f0[atomicAdd(&W.cnt, 1)] = W.cav[k];
  __syncwarp();
  const int m = W.cnt;
  DCHK(m >= 1 && m <= n);
  WMARK(50);
  if (m > O.ctet) return RS_OVERFLOW;
  int P2 = 32;
  while (P2 < m) P2 <<= 1;
  for (int k = m + lane; k < P2; k += 32) W.f0[k] = INT_MAX;
  __syncwarp();
  for (int size = 2; size <= P2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int k = lane; k < P2; k += 32) {
        int l = k ^ stride;
        if (l > k) {
          int a = W.f0[k], b = W.f0[l];
          bool up = (k & size) == 0;
          if ((a > b) == up) { W.f0[k] = b; W.f0[l] = a; }
        }
      }
      __syncwarp();
    }
  WSTOP(4);
  WMARK(14);
  // boundary faces per tet (consecutive chunks per lane keep the order)
  const int per = (m + 31) >> 5;
  const int lo = lane * per, hi = min(lo + per, m);
  int mycnt = 0;
  for (int a = lo; a < hi; ++a) {
    int t = W.f0[a];
    O.tets[a] = t;
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, t, i) >> 2;
      bool blk = blocked(D, A, t, i);
      int ku = wh_find(W, u);
      bool uin = ku >= 0 && W.in[ku];
      if (uin && !blk) continue;
      if (uin && blk) { atomicMin(&W.memb, 4 * a + i); continue; }
      ++mycnt;
    }
  }
  __syncwarp();
  DCHK(W.memb == INT_MAX || (W.memb >> 2) < m);
  if (W.memb != INT_MAX) {
    O.memb = 4 * O.tets[W.memb >> 2] + (W.memb & 3);
    if (lane == 0) atomicAdd(&D.ctr->fail[6], 1u);
    return RS_MEMBRANE;
  }
  int incl = mycnt;
  for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(FULL, incl, o); if (lane >= o) incl += v; }
  const int nbf = __shfl_sync(FULL, incl, 31);
  WMARK(50);
  if (nbf > O.cbf) return RS_OVERFLOW;
  int off = incl - mycnt;
  for (int a = lo; a < hi; ++a) {
    int t = W.f0[a];
    W.f1[a] = off;                   // first boundary face of sorted tet a
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, t, i) >> 2;
      bool blk = blocked(D, A, t, i);
      int ku = wh_find(W, u);
      bool uin = ku >= 0 && W.in[ku];
      if (uin && !blk) continue;
      O.bf[off++] = 4 * t + i;
    }
  }
  __syncwarp();
#ifndef GQ_NO_GHOSTCHECK
  // (bulk construction skips it: its hull is the convex hull of exact input points)
  if (check_ghost && W.ghost && bf_open_warp(D, O.bf, nbf, W.hkey, WR_HASH, lane)) {
    if (lane == 0) atomicAdd(&D.ctr->fail[3], 1u);
    return RS_BADSTAR;
  }
#endif
  WSTOP(5);
  WMARK(15);
  // boundary vertices: min distance and the swallow check (hash reused)
  for (int i = lane; i < WR_HASH; i += 32) W.hkey[i] = INT_MIN;
  if (lane == 0) W.flag = 0;
  __syncwarp();
  double mymin = __longlong_as_double(0x7ff0000000000000ll);
  for (int k = lane; k < nbf; k += 32) {
    int t = O.bf[k] >> 2, i = O.bf[k] & 3;
    DCHK(t >= 0 && t < D.tcap);
    int f[3]; face_verts(D.tv[t], i, f);
    for (int j = 0; j < 3; ++j) {
      if (f[j] == GHOST) continue;
      DCHK(f[j] >= 0 && f[j] < D.vcap);
      int s = wh_claim(W, f[j]);
      if (s == -2) { W.flag = 1; continue; }
      if (s < 0) continue;
      W.hval[s] = 0;
      const double* qv = PT(D, f[j]);
      double d = (qv[0] - p[0]) * (qv[0] - p[0]) + (qv[1] - p[1]) * (qv[1] - p[1]) + (qv[2] - p[2]) * (qv[2] - p[2]);
      if (d < mymin) mymin = d;
    }
  }
  for (int o = 16; o > 0; o >>= 1) { double v = __shfl_xor_sync(FULL, mymin, o); if (v < mymin) mymin = v; }
  __syncwarp();
  WMARK(50);
  if (W.flag) return RS_OVERFLOW;
  bool swallow = false;
  for (int a = lane; a < m; a += 32) {
    int4 q = D.tv[W.f0[a]];
    for (int k = 0; k < 4; ++k) {
      int v = tvk(q, k);
      if (v != GHOST && wh_find(W, v) == -1) swallow = true;
    }
  }
  WMARK(50);
  if (__any_sync(FULL, swallow)) { if (lane == 0) atomicAdd(&D.ctr->fail[2], 1u); return RS_CNSS; }
  WSTOP(6);
  WMARK(16);
  O.ntet = m; O.nbf = nbf; O.mind = mymin;
  O.ncr = 0; O.nbsub = 0; O.nbseg = 0; O.neseg = 0;
  // ---- constraint classification, warp-parallel.  Same lists and order as the
  // reference's first-met loop (_kernels.py:560-635): occurrences are listed in
  // (sorted tet, face / edge slot) order, a constraint counts at its first
  // occurrence, and a subsegment is "boundary" iff one of the boundary faces of
  // the tets up to its first one contains it (the numba partial-bedges rule).
  bool cons = false;
  for (int a = lane; a < m; a += 32) if (D.sub[W.f0[a]] || D.seg[W.f0[a]]) cons = true;
  WMARK(50);
  if (!__any_sync(FULL, cons)) return RS_OK;
  WSTOP(7);
  // occurrences: code = a << 4 | slot (slot 0-3 subface face, 4-9 subsegment edge)
  int* oc = W.hkey;                  // hkey / cav / comp / in are free after the swallow check
  int* k0 = W.cav; int* k1 = W.comp; int* k2 = W.hkey + WR_HASH / 2;
  unsigned char* ofirst = W.in;
  const int OCAP = WR_MAXT < WR_HASH / 2 ? WR_MAXT : WR_HASH / 2;
  int myocc = 0;
  for (int a = lo; a < hi; ++a) {
    int t = W.f0[a];
    myocc += __popc((unsigned)D.sub[t] & 15u) + __popc((unsigned)D.seg[t] & 63u);
  }
  int oincl = myocc;
  for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(FULL, oincl, o); if (lane >= o) oincl += v; }
  const int K = __shfl_sync(FULL, oincl, 31);
  if (K > OCAP) return RS_OVERFLOW;   // rare: the block kernel handles it
  int op = oincl - myocc;
  for (int a = lo; a < hi; ++a) {
    int t = W.f0[a];
    int4 q = D.tv[t];
    int sm = D.sub[t], em = D.seg[t];
    for (int i = 0; i < 4; ++i) {
      if (!(sm & (1 << i))) continue;
      int f[3]; face_verts(q, i, f);
      int a0 = f[0], b0 = f[1], c0 = f[2];
      sort3(a0, b0, c0);
      oc[op] = a << 4 | i; k0[op] = a0; k1[op] = b0; k2[op] = c0; ++op;
    }
    for (int i = 0; i < 6; ++i) {
      if (!(em & (1 << i))) continue;
      int x = tvk(q, c_edges[i][0]), y = tvk(q, c_edges[i][1]);
      if (x > y) { int tt = x; x = y; y = tt; }
      oc[op] = a << 4 | (4 + i); k0[op] = x; k1[op] = y; k2[op] = -1; ++op;
    }
  }
  __syncwarp();
  for (int j = lane; j < K; j += 32) {
    bool first = true;
    const bool isf = (oc[j] & 15) < 4;
    for (int i = 0; i < j && first; ++i)
      if (((oc[i] & 15) < 4) == isf && k0[i] == k0[j] && k1[i] == k1[j] && k2[i] == k2[j]) first = false;
    ofirst[j] = first;
  }
  __syncwarp();
  // subfaces: crossed (allowed and interior) or boundary, appended in order
  int st = RS_OK;
  int ncr = 0, nbs = 0;
  for (int base = 0; base < K; base += 32) {
    const int j = base + lane;
    bool isc = false, isb = false;
    int rec = -1, crf = 0;
    if (j < K && ofirst[j] && (oc[j] & 15) < 4) {
      int a = oc[j] >> 4, i = oc[j] & 15, t = W.f0[a];
      int nb = tnk(D, t, i);
      int u = nb >> 2;
      int l = 0, h = m - 1;
      bool uin = false;
      while (l <= h) { int mid = (l + h) >> 1; int v = W.f0[mid]; if (v == u) { uin = true; break; } if (v < u) l = mid + 1; else h = mid - 1; }
      rec = face_lookup(D, k0[j], k1[j], k2[j]);
      isc = uin && rec >= 0 && A.n > 0 && allowed_face(D, A, k0[j], k1[j], k2[j]);
      isb = !isc;
      crf = min(4 * t + i, nb);
    }
    unsigned bc = __ballot_sync(FULL, isc), bb = __ballot_sync(FULL, isb);
    const unsigned below = (1u << lane) - 1u;
    if (isc) { int k = ncr + __popc(bc & below); if (k < O.ccon) { O.cr[k] = rec; O.crf[k] = crf; } }
    if (isb) { int k = nbs + __popc(bb & below); if (k < O.ccon) O.bsub[k] = rec; }
    ncr += __popc(bc); nbs += __popc(bb);
  }
  if (ncr > O.ccon || nbs > O.ccon) st = RS_OVERFLOW;
  // subsegments: boundary iff an edge of the boundary faces met so far
  int nbg = 0, neg = 0;
  for (int j0 = 0; j0 < K && st == RS_OK; ++j0) {
    if (!ofirst[j0] || (oc[j0] & 15) < 4) continue;
    const int a = oc[j0] >> 4, x = k0[j0], y = k1[j0];
    const int fend = a + 1 < m ? W.f1[a + 1] : nbf;   // boundary faces of sorted tets 0..a
    bool hit = false;
    for (int k = lane; k < fend && !hit; k += 32) {
      int t = O.bf[k] >> 2, i = O.bf[k] & 3;
      int f[3]; face_verts(D.tv[t], i, f);
      bool hx = f[0] == x || f[1] == x || f[2] == x, hy = f[0] == y || f[1] == y || f[2] == y;
      hit = hx && hy;
    }
    const bool bound = __any_sync(FULL, hit);
    if (nbg + neg >= O.ccon) { st = RS_OVERFLOW; break; }
    if (lane == 0) {
      int rec = seg_lookup(D, x, y);
      if (bound) O.bseg[nbg] = rec; else O.eseg[neg] = rec;
    }
    if (bound) ++nbg; else ++neg;
  }
  O.ncr = ncr; O.nbsub = nbs; O.nbseg = nbg; O.neseg = neg;
  __syncwarp();
  WMARK(60);
  return st;
}

// The peel can remove the seed itself: on a finely split oblique surface the
// listed seed may be a nearly flat tet spanning two facet triangles whose
// faces p sees edge-on.  The reference then fails the candidate
// (_kernels.py region_kernel -> CavityNotStarShaped).  With oblique facets
// present (none of the parity inputs has one) the next listed seed in region
// is tried instead, up to three times; the peel is seed-independent, so a
// surviving seed yields the star-shaped cavity around p.
template <int MAXT, int HASH>
__device__ inline int region_warp_retry(const Dev& D, const double* p, const int* seeds, int nseeds, const Allow& A,
                                        WarpSharedT<MAXT, HASH>& W, Scratch& S, RegionOut& O) {
  unsigned excl = 0u;
  int st = RS_CNSS;
#pragma unroll 1
  for (int a = 0; a < 4; ++a) {
    st = region_warp(D, p, seeds, nseeds, A, W, S, O, true, excl, a < 3);
    if (st != RS_SHRUNK) break;
    excl |= 1u << W.seedk;
    __syncwarp();
  }
  if (st == RS_SHRUNK) st = RS_CNSS;
  return st;
}

}  // namespace gq

namespace gq {

// ---------------------------------------------------------------------------
// Warp-cooperative Bowyer-Watson star (mesh.py:736-771, _kernels.py:641-807):
// lane-parallel tet creation and outer wiring; the inner faces (those through
// the new vertex) are paired through a per-warp shared hash keyed by the edge
// of the boundary face they stand on (phase A inserts both sides, phase B
// reads the partner).  Same tets, ids and adjacency as star_insert().
#define WS_MAXF 272
#define WS_HASH 1024
#define WS_WARPS 4
struct StarShared {
  unsigned long long key[WS_HASH];
  int v0[WS_HASH];
  int v1[WS_HASH];
  int flag;
};
struct StarHash {            // view on shared (normal) or global (big cavities) storage
  unsigned long long* key;
  int* v0;
  int* v1;
  int cap;                   // power of two
  int* flag;
};

__device__ __forceinline__ int star_slot(const StarHash& X, unsigned long long key, bool insert) {
  unsigned int h = (unsigned int)mix64(key) & (X.cap - 1);
  for (int pr = 0; pr < X.cap; ++pr) {
    unsigned long long cur = X.key[h];
    if (cur == key) return (int)h;
    if (cur == EMPTY_KEY) {
      if (!insert) return -1;
      unsigned long long old = atomicCAS(&X.key[h], EMPTY_KEY, key);
      if (old == EMPTY_KEY || old == key) return (int)h;
    }
    h = (h + 1) & (X.cap - 1);
  }
  return -1;
}
__device__ __forceinline__ unsigned long long inner_key(const int* g, int vid) {
  int x = g[0] == vid ? g[1] : g[0];
  int y = g[2] == vid ? g[1] : g[2];
  if (x > y) { int tt = x; x = y; y = tt; }
  return ((unsigned long long)(unsigned int)(x + 1) << 32) | (unsigned int)(y + 1);
}

__device__ __forceinline__ StarHash star_hash_shared(StarShared& S) {
  StarHash h; h.key = S.key; h.v0 = S.v0; h.v1 = S.v1; h.cap = WS_HASH; h.flag = &S.flag; return h;
}
__device__ inline bool star_warp(const Dev& D, int vid, const int* bf, int nbf, int nt0, bool max_vt,
                                 const StarHash& X, int* touched, int stamp) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < X.cap; i += 32) { X.key[i] = EMPTY_KEY; X.v0[i] = -1; X.v1[i] = -1; }
  if (lane == 0) *X.flag = 0;
  __syncwarp();
  // phase A: new tets, outer links, inner faces into the hash
  for (int k = lane; k < nbf; k += 32) {
    int t = bf[k] >> 2, i = bf[k] & 3;
    int packed = tnk(D, t, i);
    int u = packed >> 2, j = packed & 3;
    if (touched) touched[u] = stamp;
    int f[3]; face_verts(D.tv[u], j, f);
    int nt = nt0 + k;
    int4 q;
    if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) {
      int e0, e1;
      if (f[0] == GHOST) { e0 = f[1]; e1 = f[2]; }
      else if (f[1] == GHOST) { e0 = f[2]; e1 = f[0]; }
      else { e0 = f[0]; e1 = f[1]; }
      q = make_int4(e1, e0, vid, GHOST);
    } else {
      q = make_int4(f[0], f[1], f[2], vid);
    }
    D.tv[nt] = q;
    D.alive[nt] = 1; D.skip[nt] = 0;
    int a0 = f[0], b0 = f[1], c0 = f[2];
    sort3(a0, b0, c0);
    int om = -1;
    for (int m = 0; m < 4; ++m) {
      int g[3]; face_verts(q, m, g);
      int x = g[0], y = g[1], z = g[2];
      sort3(x, y, z);
      if (om < 0 && x == a0 && y == b0 && z == c0) { om = m; continue; }
      int h = star_slot(X, inner_key(g, vid), true);
      if (h < 0) { *X.flag = 1; continue; }
      int mine = 4 * nt + m;
      if (atomicCAS(&X.v0[h], -1, mine) != -1 && atomicCAS(&X.v1[h], -1, mine) != -1) {
#ifdef GQ_DEBUG2D
        int x = g[0] == vid ? g[1] : g[0], y = g[2] == vid ? g[1] : g[2];
        printf("[star] vid %d nbf %d: edge (%d,%d) on more than two boundary faces\n", vid, nbf, x, y);
#endif
        *X.flag = 1;
      }
    }
    if (om < 0) {
#ifdef GQ_DEBUG2D
      printf("[star] vid %d nbf %d: boundary face not reproduced\n", vid, nbf);
#endif
      *X.flag = 1; continue;
    }
    set_tn(D, nt, om, 4 * u + j);
    set_tn(D, u, j, 4 * nt + om);
    for (int m = 0; m < 4; ++m) {
      int v = tvk(q, m);
      if (v == GHOST || v == vid) continue;
      if (max_vt) atomicMax(D.vert_tet + v, nt); else D.vert_tet[v] = nt;
    }
  }
  __syncwarp();
  if (*X.flag) { if (lane == 0) raise_err(GQ_ERR_STAR); return false; }
  // phase B: inner links from the partner entries
  for (int k = lane; k < nbf; k += 32) {
    int nt = nt0 + k;
    int4 q = D.tv[nt];
    for (int m = 0; m < 4; ++m) {
      int g[3]; face_verts(q, m, g);
      if (g[0] != vid && g[1] != vid && g[2] != vid) continue;   // outer face
      int h = star_slot(X, inner_key(g, vid), false);
      int mine = 4 * nt + m;
      int other = h < 0 ? -1 : (X.v0[h] == mine ? X.v1[h] : X.v0[h]);
      if (other < 0) {
#ifdef GQ_DEBUG2D
        printf("[star] vid %d nbf %d: inner face without partner\n", vid, nbf);
#endif
        *X.flag = 1; continue;
      }
      set_tn(D, nt, m, other);
    }
  }
  __syncwarp();
  if (*X.flag) { if (lane == 0) raise_err(GQ_ERR_STAR); return false; }
  for (int k = lane; k < nbf; k += 32) {
    refresh_masks(D, nt0 + k);
    star_ratio(D, nt0 + k);
  }
  __syncwarp();
  if (lane == 0) D.vert_tet[vid] = nt0;
  return true;
}

}  // namespace gq
