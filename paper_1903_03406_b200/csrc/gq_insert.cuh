// gq_insert.cuh -- insertion of the accepted set: vertices, facet retiling, stars, bookkeeping (refine.py:677-736, facets.py, mesh.py:697-816).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

// ---------------------------------------------------------------------------
// insertion of the accepted set
struct Ins {          // inserted candidates in priority order
  int* list; int n;
  int nv0, nt0base;
};

// vertex ids / points / subsegment splits (refine.py:688-708 bookkeeping)
__global__ void k_ins_vertices(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Ins I) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < I.n; k += gridDim.x * blockDim.x) {
    int c = I.list[k];
    int vid = C.vid[c];
    const double* p = C.p + 3 * (size_t)c;
    double* q = D.P + 3 * (size_t)vid;
    q[0] = p[0]; q[1] = p[1]; q[2] = p[2];
    D.vorigin[vid] = 1;
    D.vert_tet[vid] = -1;
    D.vsid[vid] = C.kind[c] == K_SEG ? D.sg_sid[C.tgt[c]] : -1;
  }
}

__device__ inline int new_seg_record(const Dev& D, int u, int v, int sid, unsigned int fl) {
  if (u > v) { int t = u; u = v; v = t; }
  int r = atomicAdd(&D.ctr->nsegrec, 1);
  if (r >= D.sgcap) { raise_err(GQ_ERR_CAP); return -1; }
  D.sg_uv[r] = make_int2(u, v); D.sg_sid[r] = sid; D.sg_fl[r] = fl;
  ht_put(D.sg_hk, D.sg_hv, D.sg_hmask, key2(u, v), r);
  return r;
}
__device__ inline int new_face_record(const Dev& D, int a, int b, int c, int pid, unsigned int fl) {
  sort3(a, b, c);
  int r = atomicAdd(&D.ctr->nfacerec, 1);
  if (r >= D.sfcap) { raise_err(GQ_ERR_CAP); return -1; }
  D.sf_v[r] = make_int4(a, b, c, pid); D.sf_fl[r] = fl;
  ht_put(D.sf_hk, D.sf_hv, D.sf_hmask, key3(a, b, c), r);
  return r;
}

// facets.py:278-291 Facet._tri_inside: a 2D triangle of the polygon's
// triangulation (which covers the convex hull of its vertices) is a subface
// iff its centroid lies inside or on the polygon (plc.py _point_in_polygon_2d),
// decided exactly: all coordinates as integers on a common power-of-two
// scale, the centroid kept as S/3 (S = a + b + c) by multiplying through by 3.
__device__ __noinline__ bool tri_in_polygon(const Dev& D, int pid, int a, int b, int c) {
  if (D.poly_convex[pid]) return true;
  const int o0 = D.poly_off[pid], n = D.poly_off[pid + 1] - o0;
  int2 kp = D.poly_keep[pid];
  auto X = [&](int v, int k) { return PT(D, v)[k == 0 ? kp.x : kp.y]; };
  int emin = 1 << 30;
  auto upd = [&](double x) { if (x != 0.0) { int e; frexp(x, &e); emin = e < emin ? e : emin; } };
  for (int k = 0; k < 2; ++k) { upd(X(a, k)); upd(X(b, k)); upd(X(c, k)); }
  for (int j = 0; j < n; ++j) for (int k = 0; k < 2; ++k) upd(X(D.poly_idx[o0 + j], k));
  if (emin == (1 << 30)) emin = 0;
  auto toBI = [&](double x, BI& r) {
    if (x == 0.0) { bi_zero(r); return; }
    int e; double m = frexp(x, &e);
    bi_set(r, (long long)(m * 9007199254740992.0), e - emin);
  };
  BI S[2], t, u, three;
  bi_set(three, 3, 0);
  for (int k = 0; k < 2; ++k) {
    BI pa, pb, pc;
    toBI(X(a, k), pa); toBI(X(b, k), pb); toBI(X(c, k), pc);
    bi_add(t, pa, pb); bi_add(S[k], t, pc);
  }
  bool inside = false;
  for (int j = 0; j < n; ++j) {
    int va = D.poly_idx[o0 + j], vb = D.poly_idx[o0 + (j + 1) % n];
    BI A[2], B[2], A3[2], d[2], w[2];
    for (int k = 0; k < 2; ++k) {
      toBI(X(va, k), A[k]); toBI(X(vb, k), B[k]);
      bi_mul(A3[k], A[k], three);
      bi_sub(d[k], B[k], A[k]);            // B - A
      bi_sub(w[k], S[k], A3[k]);           // 3 (q - A)
    }
    // on the edge: orient2d(A, B, q) == 0 and 0 <= (q-A).(B-A) <= |B-A|^2 (ends included)
    BI o1, o2, orr;
    bi_mul(o1, d[0], w[1]); bi_mul(o2, d[1], w[0]); bi_sub(orr, o1, o2);
    if (orr.s == 0) {
      BI dot, l2, p0, p1, l2x3;
      bi_mul(p0, w[0], d[0]); bi_mul(p1, w[1], d[1]); bi_add(dot, p0, p1);
      bi_mul(p0, d[0], d[0]); bi_mul(p1, d[1], d[1]); bi_add(l2, p0, p1);
      bi_mul(l2x3, l2, three);
      BI diff; bi_sub(diff, l2x3, dot);
      if (dot.s >= 0 && diff.s >= 0) return true;
    }
    // crossing number (ray towards +x): (A.y > q.y) != (B.y > q.y), then xcross > q.x
    BI B3y; bi_mul(B3y, B[1], three);
    BI da, db; bi_sub(da, A3[1], S[1]); bi_sub(db, B3y, S[1]);
    if ((da.s > 0) != (db.s > 0)) {
      BI m0, m1, N, ax3;
      bi_sub(ax3, A3[0], S[0]);            // 3 A.x - S.x
      bi_mul(m0, ax3, d[1]);               // (3Ax - Sx)(By - Ay)
      bi_mul(m1, w[1], d[0]);              // (Sy - 3Ay)(Bx - Ax)
      bi_add(N, m0, m1);
      if (N.s != 0 && N.s == d[1].s) inside = !inside;
    }
  }
  return inside;
}
__global__ void k_poly_convex(const __grid_constant__ Dev D, int f) {
  for (int pid = blockIdx.x * blockDim.x + threadIdx.x; pid < f; pid += gridDim.x * blockDim.x) {
    const int o0 = D.poly_off[pid], n = D.poly_off[pid + 1] - o0;
    int2 kp = D.poly_keep[pid];
    bool convex = true;
    for (int j = 0; j < n && convex; ++j) {
      const double *p0 = PT(D, D.poly_idx[o0 + j]), *p1 = PT(D, D.poly_idx[o0 + (j + 1) % n]),
                   *p2 = PT(D, D.poly_idx[o0 + (j + 2) % n]);
      double a2[2] = {p0[kp.x], p0[kp.y]}, b2[2] = {p1[kp.x], p1[kp.y]}, c2[2] = {p2[kp.x], p2[kp.y]};
      convex = orient2d(a2, b2, c2) >= 0;   // counterclockwise in the kept axes (facets.py:262-268)
    }
    D.poly_convex[pid] = convex ? 1 : 0;
  }
}

__global__ void k_ins_segsplit(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Ins I) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < I.n; k += gridDim.x * blockDim.x) {
    int c = I.list[k];
    if (C.kind[c] != K_SEG) continue;
    int r = C.tgt[c];
    int2 e = D.sg_uv[r];
    int sid = D.sg_sid[r];
    D.sg_fl[r] = 0;   // removed (also leaves enc_segs)
    int vid = C.vid[c];
    new_seg_record(D, e.x, vid, sid, RF_LIVE | RF_CHECK);
    new_seg_record(D, e.y, vid, sid, RF_LIVE | RF_CHECK);
  }
}

// facets.py:377-386: triangle on one segment line
__device__ __noinline__ bool collinear_sliver(const Dev& D, int a, int b, int c) {
  int v3[3] = {a, b, c};
  for (int k = 0; k < 3; ++k) {
    int s = D.vsid[v3[k]];
    if (s < 0) continue;
    int2 e = D.sid_uv[s];
    bool all = true;
    for (int j = 0; j < 3 && all; ++j) {
      int w = v3[j];
      if (D.vsid[w] == s || w == e.x || w == e.y) continue;
      all = false;
    }
    if (all) return true;
  }
  return false;
}

// 2D retiling work items: (candidate, polygon)
// per-item capacities of the facet retiling: crossed triangles of one polygon
// (local array), and 2D cavity triangles (T.cap; tri2_cavity's DFS stack and
// component marks take 2 * T.cap of the thread's 2 * Scratch.cap stack)
#define T2_FCAP 256
#define T2_CAP 512
struct T2Items {
  int* cand; int* pid; int* state; int n;   // state 0 pending, 1 done
  int* cav; int* ncav; int cap;             // per item cavity tids
  int* own;                                 // per 2D triangle owner rank
  int* rem; int* nrem; int rcap;            // removed subface records per item
  int icap;                                 // items allocated
};

__device__ __noinline__ void t2_forced(const Dev& D, const Cand& C, int c, int pid, int* forced, int& nf, int cap) {
  // crossed subfaces of this polygon (refine.py:677-683) -> their 2D triangles
  SlabView v = slab(C, c);
  nf = 0;
  for (int k = 0; k < C.ncr[c]; ++k) {
    int rec = v.cr[k];
    if (rec < 0) continue;
    int4 f = D.sf_v[rec];
    if (f.w != pid) continue;
    // triangle with directed edge a->b or b->a holding c
    int t = he_lookup(D, f.x, f.y, pid);
    if (t < 0 || !(D.t2v[t].x == f.z || D.t2v[t].y == f.z || D.t2v[t].z == f.z)) t = he_lookup(D, f.y, f.x, pid);
    if (t < 0) continue;
    if (nf < cap) forced[nf++] = t; else raise_err(GQ_ERR_CAP);   // never drop a crossed triangle silently
  }
  if (C.kind[c] == K_SEG) {   // split edge triangles (facets.py:310-315)
    int2 e = D.sg_uv[C.tgt[c]];
    int t1 = he_lookup(D, e.x, e.y, pid); if (t1 >= 0) { if (nf < cap) forced[nf++] = t1; else raise_err(GQ_ERR_CAP); }
    int t2 = he_lookup(D, e.y, e.x, pid); if (t2 >= 0) { if (nf < cap) forced[nf++] = t2; else raise_err(GQ_ERR_CAP); }
  }
}
__device__ __noinline__ int t2_seed_of(const Dev& D, const Cand& C, int c, int pid) {
  if (C.kind[c] == K_FACE) {
    int4 f = D.sf_v[C.tgt[c]];
    int t = he_lookup(D, f.x, f.y, pid);
    if (t < 0 || !(D.t2v[t].x == f.z || D.t2v[t].y == f.z || D.t2v[t].z == f.z)) t = he_lookup(D, f.y, f.x, pid);
    return t;
  }
  return -1;
}

// The passes of the facet retiling as bodies over items [start, T.n) with a
// stride: launched grid-wide for many items, or all passes fused in one block
// (k_t2_fused) when a round has few of them.
__device__ void t2_compute_body(const Dev& D, const Cand& C, const T2Items& T, Scratch& S, int start, int stride, int pm = 1, int pb = 0) {
  for (int w = start; w < T.n; w += stride) {
    if (pm > 1 && T.pid[w] % pm != pb) continue;   // another block's polygons
    if (T.state[w] != 0) continue;
    int c = T.cand[w], pid = T.pid[w];
    Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = C.vid[c]; X.follow3d = D.poly_obl[pid];
    proj2(D, pid, C.p + 3 * (size_t)c, X.p);
    int forced[T2_FCAP + 1]; int nf;      // the crossed triangles, then (seeds) the target's own
    t2_forced(D, C, c, pid, forced, nf, T2_FCAP);
    const int* seeds = forced; int ns = nf;
    int ts = t2_seed_of(D, C, c, pid);
    if (ts >= 0) forced[ns++] = ts;
    int n = tri2_cavity(X, forced, nf, seeds, ns, S.tset, T.cav + (size_t)w * T.cap, S.stack, T.cap);
    if (n < 0) {
#ifdef GQ_DEBUG2D
      printf("[2d] cavity fail pid %d vid %d\n", pid, X.vid);
#endif
      raise_err(GQ_ERR_2D); n = 0;
    }
    T.ncav[w] = n;
  }
}
template <class F>
__device__ inline void t2_for_claims(const Dev& D, const T2Items& T, int w, F f) {
  const int* cav = T.cav + (size_t)w * T.cap;
  int pid = T.pid[w];
  for (int k = 0; k < T.ncav[w]; ++k) {
    int tid = cav[k];
    f(tid);
    int4 t = D.t2v[tid];
    for (int e = 0; e < 3; ++e) { int nb = t2_nb(D, t, e); if (nb >= 0) f(nb); }
    (void)pid;
  }
}
__device__ void t2_claim_body(const Dev& D, const Cand& C, const T2Items& T, int start, int stride, int pm = 1, int pb = 0) {
  for (int w = start; w < T.n; w += stride) {
    if (pm > 1 && T.pid[w] % pm != pb) continue;   // another block's polygons
    if (T.state[w] != 0) continue;
    int r = C.rank[T.cand[w]];
    t2_for_claims(D, T, w, [&](int tid) { atomicMin(T.own + tid, r); });
  }
}
__device__ void t2_apply_body(const Dev& D, const Cand& C, const T2Items& T, int* applied, int start, int stride, int pm = 1, int pb = 0) {
  for (int w = start; w < T.n; w += stride) {
    if (pm > 1 && T.pid[w] % pm != pb) continue;   // another block's polygons
    if (T.state[w] != 0) continue;
    int c = T.cand[w];
    int r = C.rank[c];
    bool win = true;
    t2_for_claims(D, T, w, [&](int tid) { if (T.own[tid] != r) win = false; });
    if (!win) continue;
    T.state[w] = 2;   // apply (owners reset next)
    atomicAdd(applied, 1);
  }
}
__device__ void t2_commit_body(const Dev& D, const Cand& C, const T2Items& T, Scratch& S, int start, int stride, int pm = 1, int pb = 0) {
  for (int w = start; w < T.n; w += stride) {
    if (pm > 1 && T.pid[w] % pm != pb) continue;   // another block's polygons
    if (T.state[w] != 2) continue;
    int c = T.cand[w], pid = T.pid[w];
    Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = C.vid[c]; X.follow3d = D.poly_obl[pid];
    proj2(D, pid, C.p + 3 * (size_t)c, X.p);
    int n = T.ncav[w];
    int* cav = T.cav + (size_t)w * T.cap;
    S.tset.clear();
    for (int k = 0; k < n; ++k) S.tset.put(cav[k], k);
    int* rem = T.rem + (size_t)w * T.rcap;
    int nrem = 0;
    tri2_apply(X, cav, n, S.tset,
      [&](int a, int b, int cc) {          // removed: rem &= keys_by_pid
        sort3(a, b, cc);
        int rec = face_lookup(D, a, b, cc);
        if (rec >= 0 && D.sf_v[rec].w == pid) {
          if (nrem < T.rcap) rem[nrem++] = rec; else raise_err(GQ_ERR_CAP);
        }
      },
      [&](int a, int b, int cc, int t2) {  // added, unless a collinear sliver or outside the polygon
        if (collinear_sliver(D, a, b, cc)) return;
        if (!tri_in_polygon(D, pid, a, b, cc)) return;
        int a0 = a, b0 = b, c0 = cc; sort3(a0, b0, c0);
        if (face_lookup(D, a0, b0, c0) >= 0) return;   // never add a key twice
        new_face_record(D, a0, b0, c0, pid, RF_LIVE | RF_CHECK);
      });
    T.nrem[w] = nrem;
    T.state[w] = 1;
  }
}
__device__ void t2_reset_body(const Dev& D, const T2Items& T, int final_pass, int start, int stride, int pm = 1, int pb = 0) {
  for (int w = start; w < T.n; w += stride) {
    if (pm > 1 && T.pid[w] % pm != pb) continue;   // another block's polygons
    if (!final_pass && T.state[w] == 1 && T.ncav[w] < 0) continue;
    t2_for_claims(D, T, w, [&](int tid) { T.own[tid] = INT_MAX; });
  }
}
// retire the removed subface records (after every pass, so lookups in later
// passes still see the pre-round tables only for untouched keys)
__device__ void t2_retire_body(const Dev& D, const T2Items& T, int start, int stride, int pm = 1, int pb = 0) {
  for (int w = start; w < T.n; w += stride) {
    if (pm > 1 && T.pid[w] % pm != pb) continue;   // another block's polygons
    const int* rem = T.rem + (size_t)w * T.rcap;
    for (int k = 0; k < T.nrem[w]; ++k) D.sf_fl[rem[k]] = 0;
  }
}

#define GRID_START (blockIdx.x * blockDim.x + threadIdx.x)
#define GRID_STRIDE (gridDim.x * blockDim.x)
__global__ void k_t2_compute(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, const __grid_constant__ Scr SC) {
  Scratch S = scratch_for(SC, GRID_START);
  t2_compute_body(D, C, T, S, GRID_START, GRID_STRIDE);
}
__global__ void k_t2_claim(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T) { t2_claim_body(D, C, T, GRID_START, GRID_STRIDE); }
__global__ void k_t2_apply(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, const __grid_constant__ Scr SC, int* applied) { t2_apply_body(D, C, T, applied, GRID_START, GRID_STRIDE); }
__global__ void k_t2_commit(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, const __grid_constant__ Scr SC) {
  Scratch S = scratch_for(SC, GRID_START);
  t2_commit_body(D, C, T, S, GRID_START, GRID_STRIDE);
}
__global__ void k_t2_reset(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, int final_pass) { t2_reset_body(D, T, final_pass, GRID_START, GRID_STRIDE); }
__global__ void k_t2_retire(const __grid_constant__ Dev D, T2Items T) { t2_retire_body(D, T, GRID_START, GRID_STRIDE); }
// One item per warp on lane 0: an item is a long chain of dependent hash and
// mesh loads whose trip counts differ item to item, so items sharing a warp
// serialise each other's divergent paths; alone in a warp they only wait on
// memory, which the other resident warps hide (C5: 2D passes 3x faster).
#define WARP_ITEM_START ((int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5))
#define WARP_ITEM_STRIDE ((int)((gridDim.x * blockDim.x) >> 5))
__global__ void k_t2w_compute(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, const __grid_constant__ Scr SC) {
  if (threadIdx.x & 31) return;
  Scratch S = scratch_for(SC, WARP_ITEM_START);
  t2_compute_body(D, C, T, S, WARP_ITEM_START, WARP_ITEM_STRIDE);
}
__global__ void k_t2w_claim(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T) { if (!(threadIdx.x & 31)) t2_claim_body(D, C, T, WARP_ITEM_START, WARP_ITEM_STRIDE); }
__global__ void k_t2w_apply(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, int* applied) {
  if (!(threadIdx.x & 31)) t2_apply_body(D, C, T, applied, WARP_ITEM_START, WARP_ITEM_STRIDE);
}
__global__ void k_t2w_reset(const __grid_constant__ Dev D, T2Items T, int final_pass) { if (!(threadIdx.x & 31)) t2_reset_body(D, T, final_pass, WARP_ITEM_START, WARP_ITEM_STRIDE); }
__global__ void k_t2w_commit(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, const __grid_constant__ Scr SC) {
  if (threadIdx.x & 31) return;
  Scratch S = scratch_for(SC, WARP_ITEM_START);
  t2_commit_body(D, C, T, S, WARP_ITEM_START, WARP_ITEM_STRIDE);
}

// every pass of a round without launches or host reads between passes.  The
// items of different polygons never share a 2D triangle, so block b takes the
// polygons with pid % gridDim.x == b and runs its own passes.
// WARP: one item per warp (lane 0) as in the multi-launch passes
template <bool WARP>
__global__ void __launch_bounds__(256) k_t2_fused(const __grid_constant__ Dev D, const __grid_constant__ Cand C, T2Items T, const __grid_constant__ Scr SC, int* applied_total) {
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
  Scratch S = scratch_for(SC, WARP ? blockIdx.x * nw + wid : blockIdx.x * blockDim.x + threadIdx.x);
  const int pm = gridDim.x, pb = blockIdx.x;
  const int i0 = WARP ? ((threadIdx.x & 31) ? T.n : wid) : threadIdx.x, di = WARP ? nw : blockDim.x;
  __shared__ int s_applied, s_left;
  if (threadIdx.x == 0) s_left = 0;
  __syncthreads();
  int mine = 0;
  for (int w = threadIdx.x; w < T.n; w += blockDim.x) mine += (T.pid[w] % pm == pb);
  atomicAdd(&s_left, mine);
  __syncthreads();
  int left = s_left;
  const int total = left;
  for (int pass = 0; left > 0; ++pass) {
    if (threadIdx.x == 0) s_applied = 0;
    t2_compute_body(D, C, T, S, i0, di, pm, pb);
    __syncthreads();
    t2_claim_body(D, C, T, i0, di, pm, pb);
    __syncthreads();
    t2_apply_body(D, C, T, &s_applied, i0, di, pm, pb);
    __syncthreads();
    t2_reset_body(D, T, 1, i0, di, pm, pb);
    __syncthreads();
    t2_commit_body(D, C, T, S, i0, di, pm, pb);
    __syncthreads();
    t2_retire_body(D, T, threadIdx.x, blockDim.x, pm, pb);
    __syncthreads();
    const int applied = s_applied;
    __syncthreads();
    if (applied == 0) { if (threadIdx.x == 0) raise_err(GQ_ERR_2D); break; }
    left -= applied;
  }
  if (threadIdx.x == 0) atomicAdd(applied_total, total - left);
}

__global__ void k_kill_cavities(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Ins I) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < I.n; k += gridDim.x * blockDim.x) {
    int c = I.list[k];
    SlabView v = slab(C, c);
    for (int j = 0; j < C.ntet[c]; ++j) D.alive[v.tets[j]] = 0;
  }
}
__global__ void k_star(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Ins I) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < I.n; k += gridDim.x * blockDim.x) {
    int c = I.list[k];
    SlabView v = slab(C, c);
    star_insert(D, C.vid[c], v.bf, C.nbf[c], C.nt0[c], true);
  }
}
// warp per inserted cavity (serial star for oversized boundaries)
// global-memory pairing hash for stars of oversized cavities: the big
// scratch arena of warp gw % SB.nthreads (keys: fkey, partners: tkey/tval)
__device__ inline StarHash big_star_hash(const Scr& SB, int gw, int* flag) {
  int slot = gw % SB.nthreads;
  StarHash h;
  h.key = SB.fkey + (size_t)slot * SB.fcap;
  h.v0 = SB.tkey + (size_t)slot * SB.tcap;
  h.v1 = SB.tval + (size_t)slot * SB.tcap;
  h.cap = SB.tcap < SB.fcap ? SB.tcap : SB.fcap;
  h.flag = flag;
  return h;
}
__device__ inline StarHash huge_star_hash(const Cand& C, int c, int* flag) {
  size_t h = (size_t)(C.bigi[c] - HUGE_BASE) * C.hs;
  StarHash X;
  X.key = C.hskey + h; X.v0 = C.hsv0 + h; X.v1 = C.hsv1 + h; X.cap = C.hs; X.flag = flag;
  return X;
}
__global__ void __launch_bounds__(32 * WS_WARPS) k_star_warp(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Ins I, const __grid_constant__ Scr SB) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StarShared& X = reinterpret_cast<StarShared*>(smem_raw)[wib];
  const int gw = blockIdx.x * WS_WARPS + wib, nw = gridDim.x * WS_WARPS;
  unsigned long long n_created = 0, n_deleted = 0;
  for (int k = gw; k < I.n; k += nw) {
    int c = I.list[k];
    SlabView v = slab(C, c);
    int nbf = C.nbf[c];
    if (nbf <= WS_MAXF) star_warp(D, C.vid[c], v.bf, nbf, C.nt0[c], true, star_hash_shared(X), nullptr, 0);
    else if (C.bigi[c] >= HUGE_BASE) star_warp(D, C.vid[c], v.bf, nbf, C.nt0[c], true, huge_star_hash(C, c, &X.flag), nullptr, 0);
    else star_warp(D, C.vid[c], v.bf, nbf, C.nt0[c], true, big_star_hash(SB, gw, &X.flag), nullptr, 0);
    if (lane == 0) { n_created += nbf; n_deleted += C.ntet[c]; }
    __syncwarp();
  }
  if (lane == 0 && n_created) { atomicAdd(&D.ctr->created, n_created); atomicAdd(&D.ctr->deleted, n_deleted); }
}
__global__ void __launch_bounds__(32 * WS_WARPS) k_init_stars_warp(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* pend, const int* plist,
                                                                   const int* acc, int nw_, int* touched, int round, const __grid_constant__ Scr SB) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StarShared& X = reinterpret_cast<StarShared*>(smem_raw)[wib];
  const int gw = blockIdx.x * WS_WARPS + wib, nw = gridDim.x * WS_WARPS;
  unsigned long long n_created = 0, n_deleted = 0;
  for (int w = gw; w < nw_; w += nw) {
    if (!acc[w]) continue;
    int c = plist[w];
    SlabView v = slab(C, c);
    int nbf = C.nbf[c];
    if (nbf <= WS_MAXF) star_warp(D, pend[c], v.bf, nbf, C.nt0[c], true, star_hash_shared(X), touched, round);
    else star_warp(D, pend[c], v.bf, nbf, C.nt0[c], true, big_star_hash(SB, gw, &X.flag), touched, round);
    if (lane == 0) { n_created += nbf; n_deleted += C.ntet[c]; }
    __syncwarp();
    if (lane == 0) C.status[c] = CS_DROP;
  }
  if (lane == 0 && n_created) { atomicAdd(&D.ctr->created, n_created); atomicAdd(&D.ctr->deleted, n_deleted); }
}

// dirty constraints + survivor mask refresh for subfaces retiled in 2D but
// not crossed by the 3D cavity (refine.py:720-736)
__global__ void k_post_insert(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Ins I, T2Items T, const __grid_constant__ Scr SC, const int* item_of) {
  int tid0 = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid0);
  for (int k = tid0; k < I.n; k += gridDim.x * blockDim.x) {
    int c = I.list[k];
    SlabView v = slab(C, c);
    for (int j = 0; j < C.nbsub[c]; ++j) { int r = v.bsub[j]; if (r >= 0) atomicOr(D.sf_fl + r, D.sf_fl[r] & RF_LIVE ? RF_CHECK : 0u); }
    for (int j = 0; j < C.nbseg[c]; ++j) { int r = v.bseg[j]; if (r >= 0) atomicOr(D.sg_fl + r, D.sg_fl[r] & RF_LIVE ? RF_CHECK : 0u); }
    if (C.kind[c] == K_TET || !item_of) continue;
    for (int w = item_of[2 * k]; w < item_of[2 * k + 1]; ++w) {
      const int* rem = T.rem + (size_t)w * T.rcap;
      for (int j = 0; j < T.nrem[w]; ++j) {
        int rec = rem[j];
        bool crossed = false;
        for (int q = 0; q < C.ncr[c]; ++q) if (v.cr[q] == rec) { crossed = true; break; }
        if (crossed) continue;
        int4 f = D.sf_v[rec];
        int slot = find_face(D, f.x, f.y, f.z, S.tset, S.stack, 2 * S.cap);
        if (slot >= 0) {
          int t = slot >> 2;
          refresh_masks(D, t);
          int u = tnk(D, t, slot & 3) >> 2;
          if (u >= 0 && D.alive[u]) refresh_masks(D, u);
        }
      }
    }
  }
}

