// gq_block.cuh -- block-cooperative Delaunay region for oversized cavities.
//
// Same decisions as region_compute() (mesh.py:450-521 / _kernels.py:392-635),
// but one 256-thread block works on one cavity: the grown set lives in a
// shared-memory hash, growth is a level-synchronous frontier, the confluent
// peel and the seed component run as parallel passes, the cavity is sorted
// by tet id with a block bitonic sort and boundary faces are written in the
// reference order through a block scan.  Constraint bookkeeping (subface /
// subsegment classification, whose "first met" rule is order dependent)
// stays a serial pass of thread 0 over the sorted cavity.
#pragma once
#include "gq_dev.cuh"

namespace gq {

#define BR_THREADS 256
#define BR_MAXT 4096        // cavity tets (== CTB)
#define BR_HASH 8192

// Storage of the normal tier (dynamic shared memory).  region_block works on a
// BlockView -- pointers to the arrays plus the shared scalars -- so the same
// code also runs on global-memory arrays of any capacity (the huge tier:
// cavities of box corners or far circumcentres, tens of thousands of tets).
struct BlockShared {
  int hkey[BR_HASH];
  int hval[BR_HASH];
  int cav[BR_MAXT];
  int f0[BR_MAXT];
  int f1[BR_MAXT];
  uint8_t in[BR_MAXT];
  int comp[BR_MAXT];
};
struct BlockView {             // lives in __shared__ memory (scalars shared by the block)
  int* hkey; int* hval; int* cav; int* f0; int* f1; uint8_t* in; int* comp;
  int hcap, mcap;              // hash slots (power of two) / cavity tets
  int n, nf0, nf1, seed, status, flag, memb, cnt;
  unsigned long long mind;
};
__device__ inline void view_of_shared(BlockView& V, BlockShared& S) {
  V.hkey = S.hkey; V.hval = S.hval; V.cav = S.cav; V.f0 = S.f0; V.f1 = S.f1; V.in = S.in; V.comp = S.comp;
  V.hcap = BR_HASH; V.mcap = BR_MAXT;
}

__device__ __forceinline__ unsigned int bh(int k, int hcap) { return ((unsigned int)k * 2654435761u) & (unsigned int)(hcap - 1); }
// claim key k; returns slot if this call inserted it, -1 if present, -2 if full
__device__ inline int bh_claim(BlockView& B, int k) {
  unsigned int i = bh(k, B.hcap);
  for (int p = 0; p < B.hcap; ++p) {
    int cur = B.hkey[i];
    if (cur == k) return -1;
    if (cur == INT_MIN) {
      int old = atomicCAS(&B.hkey[i], INT_MIN, k);
      if (old == INT_MIN) return (int)i;
      if (old == k) return -1;
    }
    i = (i + 1) & (unsigned int)(B.hcap - 1);
  }
  return -2;
}
__device__ inline int bh_find(const BlockView& B, int k) {
  unsigned int i = bh(k, B.hcap);
  for (int p = 0; p < B.hcap; ++p) {
    int cur = B.hkey[i];
    if (cur == k) return B.hval[i];
    if (cur == INT_MIN) return -1;
    i = (i + 1) & (unsigned int)(B.hcap - 1);
  }
  return -1;
}

// Requires blockDim.x == BR_THREADS.  Writes O like region_compute; S is the
// block's global scratch (used only by thread 0 for the constraint pass).
__device__ inline int region_block(const Dev& D, const double* p, const int* seeds, int nseeds, const Allow& A,
                                   BlockView& B, Scratch& S, RegionOut& O) {
  int tid = threadIdx.x;
  for (int i = tid; i < B.hcap; i += BR_THREADS) B.hkey[i] = INT_MIN;
  if (tid == 0) {
    B.status = RS_OK; B.flag = 0; B.memb = INT_MAX; B.n = 0;
    int seed = -1;
    int cands[32];
    int nc = nseeds < 32 ? nseeds : 32;
    for (int k = 0; k < nc; ++k) cands[k] = seeds[k];
    bool walked = false;
    while (true) {
      seed = -1;
      for (int k = 0; k < nc; ++k) {
        int t = cands[k];
        if (t < 0 || !D.alive[t]) continue;
        if (in_region(D, t, p, A)) { seed = t; break; }
      }
      if (seed >= 0 || walked) break;
      walked = true;
      int t = walk(D, p, nc > 0 ? cands[0] : -1);
      if (t < 0) break;
      cands[0] = t; nc = 1;
    }
    B.seed = seed;
    if (seed < 0) B.status = RS_CNSS;
  }
  __syncthreads();
  if (B.status != RS_OK) return B.status;
  if (tid == 0) {
    int s = bh_claim(B, B.seed);
    if (s >= 0) B.hval[s] = 0;
    B.cav[0] = B.seed; B.n = 1;
    B.f0[0] = B.seed; B.nf0 = 1;
  }
  __syncthreads();
  O.seed = B.seed;
  // ---- grow: level-synchronous frontier
  int* cur = B.f0; int* nxt = B.f1;
  int ncur = 1;
  while (ncur > 0) {
    if (tid == 0) B.nf1 = 0;
    __syncthreads();
    for (int j = tid; j < 4 * ncur; j += BR_THREADS) {
      int t = cur[j >> 2], i = j & 3;
      int u = tnk(D, t, i) >> 2;
      if (u < 0 || !D.alive[u]) continue;
      if (blocked(D, A, t, i)) continue;
      int slot = bh_claim(B, u);
      if (slot == -1) continue;
      if (slot == -2) { B.flag = 1; continue; }
      if (in_region(D, u, p, A)) {
        int idx = atomicAdd(&B.n, 1);
        if (idx >= B.mcap) { B.flag = 1; B.hval[slot] = -2; continue; }
        B.cav[idx] = u;
        B.hval[slot] = idx;
        int q = atomicAdd(&B.nf1, 1);
        nxt[q] = u;
      } else {
        B.hval[slot] = -2;
      }
    }
    __syncthreads();
    if (B.flag) return RS_OVERFLOW;
    ncur = B.nf1;
    int* tmp = cur; cur = nxt; nxt = tmp;
    __syncthreads();
  }
  int n = B.n;
  // ---- peel + seed component (confluent; parallel passes converge to the same set)
  for (int k = tid; k < n; k += BR_THREADS) B.in[k] = 1;
  __syncthreads();
  while (true) {
    while (true) {
      if (tid == 0) B.cnt = 0;
      __syncthreads();
      for (int k = tid; k < n; k += BR_THREADS) {
        if (!B.in[k]) continue;
        int t = B.cav[k];
        int4 q = D.tv[t];
        for (int i = 0; i < 4; ++i) {
          int u = tnk(D, t, i) >> 2;
          bool blk = blocked(D, A, t, i);
          int ku = bh_find(B, u);
          bool uin = ku >= 0 && B.in[ku];
          if (uin && !blk) continue;
          int f[3]; face_verts(q, i, f);
          if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) continue;
          if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) >= 0) { B.in[k] = 0; B.cnt = 1; break; }
        }
      }
      __syncthreads();
      int ch = B.cnt;
      __syncthreads();
      if (!ch) break;
    }
    if (!B.in[0]) return RS_CNSS;       // seed shrunk away (cav[0] == seed)
    // component of the seed through unblocked faces
    for (int k = tid; k < n; k += BR_THREADS) B.comp[k] = 0;
    __syncthreads();
    if (tid == 0) { B.comp[0] = 1; B.f0[0] = 0; B.nf0 = 1; B.cnt = 1; }
    __syncthreads();
    int* fa = B.f0; int* fb = B.f1;
    int nfa = 1;
    while (nfa > 0) {
      if (tid == 0) B.nf1 = 0;
      __syncthreads();
      for (int j = tid; j < 4 * nfa; j += BR_THREADS) {
        int k = fa[j >> 2], i = j & 3;
        int t = B.cav[k];
        int u = tnk(D, t, i) >> 2;
        int ku = bh_find(B, u);
        if (ku < 0 || !B.in[ku]) continue;
        if (blocked(D, A, t, i)) continue;
        if (atomicCAS(&B.comp[ku], 0, 1) != 0) continue;
        atomicAdd(&B.cnt, 1);
        int q = atomicAdd(&B.nf1, 1);
        fb[q] = ku;
      }
      __syncthreads();
      nfa = B.nf1;
      int* tmp = fa; fa = fb; fb = tmp;
      __syncthreads();
    }
    int live = 0;
    for (int k = tid; k < n; k += BR_THREADS) live += B.in[k];
    // block sum via atomics on a shared counter
    __shared__ int s_live;
    if (tid == 0) s_live = 0;
    __syncthreads();
    atomicAdd(&s_live, live);
    __syncthreads();
    int ncomp = B.cnt;
    bool done = ncomp == s_live;
    __syncthreads();
    if (done) break;
    for (int k = tid; k < n; k += BR_THREADS) B.in[k] = B.comp[k];
    __syncthreads();
  }
  // ---- finish: sorted cavity (bitonic sort of tet ids, padded with INT_MAX)
  __shared__ int s_m;
  if (tid == 0) s_m = 0;
  __syncthreads();
  for (int k = tid; k < n; k += BR_THREADS) if (B.in[k]) { int q = atomicAdd(&s_m, 1); B.f0[q] = B.cav[k]; }
  __syncthreads();
  int m = s_m;
  if (m > O.ctet) return RS_OVERFLOW;
  int P2 = 1;
  while (P2 < m) P2 <<= 1;
  for (int k = m + tid; k < P2; k += BR_THREADS) B.f0[k] = INT_MAX;
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int k = tid; k < P2; k += BR_THREADS) {
        int l = k ^ stride;
        if (l > k) {
          int a = B.f0[k], b = B.f0[l];
          bool up = (k & size) == 0;
          if ((a > b) == up) { B.f0[k] = b; B.f0[l] = a; }
        }
      }
      __syncthreads();
    }
  }
  // re-index: hash value -> sorted position for members (needed by the serial
  // constraint pass); boundary-face counts per tet
  for (int a = tid; a < m; a += BR_THREADS) {
    int t = B.f0[a];
    O.tets[a] = t;
    int4 q = D.tv[t];
    int cnt = 0;
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, t, i) >> 2;
      bool blk = blocked(D, A, t, i);
      int ku = bh_find(B, u);
      bool uin = ku >= 0 && B.in[ku];
      if (uin && !blk) continue;
      if (uin && blk) { atomicMin(&B.memb, 4 * a + i); continue; }
      ++cnt;
    }
    (void)q;
    B.f1[a] = cnt;
  }
  __syncthreads();
  if (B.memb != INT_MAX) { O.memb = 4 * O.tets[B.memb >> 2] + (B.memb & 3); return RS_MEMBRANE; }
  // exclusive scan of f1[0..m) (serial chunks + block prefix)
  __shared__ int s_part[BR_THREADS];
  int per = (m + BR_THREADS - 1) / BR_THREADS;
  int lo = tid * per, hi = lo + per < m ? lo + per : m;
  int sum = 0;
  for (int a = lo; a < hi; ++a) sum += B.f1[a];
  s_part[tid] = sum;
  __syncthreads();
  if (tid == 0) { int acc = 0; for (int k = 0; k < BR_THREADS; ++k) { int v = s_part[k]; s_part[k] = acc; acc += v; } B.cnt = acc; }
  __syncthreads();
  int nbf = B.cnt;
  if (nbf > O.cbf) return RS_OVERFLOW;
  int off = s_part[tid];
  for (int a = lo; a < hi; ++a) {
    int t = B.f0[a];
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, t, i) >> 2;
      bool blk = blocked(D, A, t, i);
      int ku = bh_find(B, u);
      bool uin = ku >= 0 && B.in[ku];
      if (uin && !blk) continue;
      O.bf[off++] = 4 * t + i;
    }
  }
  __syncthreads();
  if (__syncthreads_or(bf_has_ghost_part(D, O.bf, nbf, tid, BR_THREADS)) &&
      bf_open_block(D, O.bf, nbf, S.fset, BR_THREADS))
    return RS_BADSTAR;
  // swallow check + min distance over boundary vertices: reuse the hash as a
  // vertex set (cavity membership is no longer needed)
  for (int i = tid; i < B.hcap; i += BR_THREADS) B.hkey[i] = INT_MIN;
  if (tid == 0) { B.mind = 0x7ff0000000000000ull; B.flag = 0; }
  __syncthreads();
  unsigned long long my = 0x7ff0000000000000ull;
  for (int k = tid; k < nbf; k += BR_THREADS) {
    int t = O.bf[k] >> 2, i = O.bf[k] & 3;
    int f[3]; face_verts(D.tv[t], i, f);
    for (int j = 0; j < 3; ++j) {
      if (f[j] == GHOST) continue;
      int s = bh_claim(B, f[j]);
      if (s == -2) { B.flag = 1; continue; }
      if (s < 0) continue;
      B.hval[s] = 0;
      const double* qv = PT(D, f[j]);
      double d = (qv[0] - p[0]) * (qv[0] - p[0]) + (qv[1] - p[1]) * (qv[1] - p[1]) + (qv[2] - p[2]) * (qv[2] - p[2]);
      unsigned long long b = (unsigned long long)__double_as_longlong(d);
      if (b < my) my = b;
    }
  }
  atomicMin(&B.mind, my);
  __syncthreads();
  if (B.flag) return RS_OVERFLOW;
  for (int a = tid; a < m; a += BR_THREADS) {
    int4 q = D.tv[B.f0[a]];
    for (int k = 0; k < 4; ++k) {
      int v = tvk(q, k);
      if (v != GHOST && bh_find(B, v) == -1) B.flag = 2;
    }
  }
  __syncthreads();
  if (B.flag == 2) return RS_CNSS;        // swallows a vertex
  O.ntet = m; O.nbf = nbf; O.mind = __longlong_as_double((long long)B.mind);
  O.ncr = 0; O.nbsub = 0; O.nbseg = 0; O.neseg = 0;
  // ---- constraint classification (order dependent; serial, thread 0)
  __shared__ int s_cons;
  if (tid == 0) s_cons = 0;
  __syncthreads();
  for (int a = tid; a < m; a += BR_THREADS) if (D.sub[B.f0[a]] || D.seg[B.f0[a]]) s_cons = 1;
  __syncthreads();
  if (!s_cons) return RS_OK;
  if (tid == 0) {
    // thread 0, first-met order (_kernels.py:560-635).  Cavity membership by
    // binary search in the sorted cavity; the boundary-edge set (needed only
    // to classify subsegments) is built lazily, up to the current tet, the
    // first time a subsegment is met.
    S.fset.clear();
    auto member = [&](int u) {
      int l = 0, h = m - 1;
      while (l <= h) { int mid = (l + h) >> 1; int v = B.f0[mid]; if (v == u) return true; if (v < u) l = mid + 1; else h = mid - 1; }
      return false;
    };
    const unsigned long long TE = 2ull << 60, TSF = 3ull << 60, TSG = 4ull << 60;
    int st = RS_OK;
    int te_upto = 0;       // boundary faces O.bf[0..te_upto) are in the edge set
    int bf_end = 0;        // boundary faces of sorted tets 0..a
    for (int a = 0; a < m && st == RS_OK; ++a) {
      int t = B.f0[a];
      int4 q = D.tv[t];
      bf_end += B.f1[a];
      int sm = D.sub[t];
      for (int i = 0; sm && i < 4; ++i) {
        if (!(sm & (1 << i))) continue;
        int f[3]; face_verts(q, i, f);
        int a0 = f[0], b0 = f[1], c0 = f[2];
        sort3(a0, b0, c0);
        int ins = S.fset.add(TSF | (key3(a0, b0, c0) & ((1ull << 60) - 1)));
        if (ins < 0) { st = RS_OVERFLOW; break; }
        if (ins == 0) continue;
        bool uin = member(tnk(D, t, i) >> 2);
        int rec = face_lookup(D, a0, b0, c0);
        bool crossed = uin && rec >= 0 && A.n > 0 && allowed_face(D, A, a0, b0, c0);
        if (crossed) {
          if (O.ncr >= O.ccon) { st = RS_OVERFLOW; break; }
          O.cr[O.ncr] = rec; O.crf[O.ncr] = min(4 * t + i, tnk(D, t, i)); O.ncr++;
        } else {
          if (O.nbsub >= O.ccon) { st = RS_OVERFLOW; break; }
          O.bsub[O.nbsub++] = rec;
        }
      }
      int em = D.seg[t];
      for (int i = 0; em && i < 6 && st == RS_OK; ++i) {
        if (!(em & (1 << i))) continue;
        int x = tvk(q, c_edges[i][0]), y = tvk(q, c_edges[i][1]);
        if (x > y) { int tt = x; x = y; y = tt; }
        int ins = S.fset.add(TSG | ((unsigned long long)x << 30) | (unsigned long long)y);
        if (ins < 0) { st = RS_OVERFLOW; break; }
        if (ins == 0) continue;
        for (; te_upto < bf_end && st == RS_OK; ++te_upto) {   // catch the edge set up to tet a
          int bt = O.bf[te_upto] >> 2, bi = O.bf[te_upto] & 3;
          int f[3]; face_verts(D.tv[bt], bi, f);
          for (int k = 0; k < 3; ++k) {
            int u = f[k], w = f[(k + 1) % 3];
            if (u == GHOST || w == GHOST) continue;
            if (u > w) { int tt = u; u = w; w = tt; }
            if (S.fset.add(TE | ((unsigned long long)u << 30) | (unsigned long long)w) < 0) st = RS_OVERFLOW;
          }
        }
        int rec = seg_lookup(D, x, y);
        bool bound = S.fset.has(TE | ((unsigned long long)x << 30) | (unsigned long long)y);
        if (O.nbseg + O.neseg >= O.ccon) { st = RS_OVERFLOW; break; }
        if (bound) O.bseg[O.nbseg++] = rec; else O.eseg[O.neseg++] = rec;
      }
    }
    B.status = st;
  }
  __syncthreads();
  return B.status;
}

}  // namespace gq
