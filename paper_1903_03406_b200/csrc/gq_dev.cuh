// gq_dev.cuh -- GPU-resident constrained tetrahedral mesh and the
// per-candidate device routines of gQM3D refinement.
//
// Layout (all SoA in HBM, 32-bit ids):
//   vertices  P[3*v] f64, vorigin u8, vert_tet i32, vsid i32 (segment of a
//             segment Steiner point, for the collinear-sliver rule)
//   tets      tv int4 (ghost = -1 in slot 3), tn int4 packed 4*t+f,
//             alive/sub/seg/skip u8, ratio f64
//   subsegments   records {u,v} sid flags  + open-addressing hash (u,v)->rec
//   subfaces      records {a,b,c,pid} flags + hash (a,b,c)->rec
//   facet 2D triangulations  t2v int4 {a,b,c,pid} (ghost -1 in slot 2),
//             t2alive u8 + half-edge hash (a,b,pid)->triangle
// Conventions follow /root/reference/pkg/src/tetrefine/mesh.py:9-18, 40-46.
#pragma once
#include "gq_exact.cuh"

namespace gq {

#define GHOST (-1)
__constant__ int c_faces[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};
__constant__ int c_edges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

// record flags
#define RF_LIVE 1u
#define RF_ENC 2u
#define RF_SKIP 4u
#define RF_BLOCK 8u
#define RF_CHECK 16u
#define RF_REDIR 32u
#define RF_FOUND 64u

#define EMPTY_KEY 0xffffffffffffffffull

struct Counters {
  int nv, nt, nsegrec, nfacerec, nt2;
  int nskip;
  int ncand;
  int pad;
  int line_pad[24];                  // the hot counts above own their 128-byte line (the
                                     // instrumentation atomics below must not share it)
  // instrumentation (SURVEY 8(d) algorithmic bytes), per context
  unsigned long long region_calls;   // region computations
  unsigned long long tested;         // tets tested for membership (cavity + boundary neighbours)
  unsigned long long cands;          // refinement candidates constructed (N_cand)
  unsigned long long claims;         // claim keys of the candidates entering a filter (K_claims)
  unsigned long long created;        // tets created by stars, bulk construction included (T_created)
  unsigned long long deleted;        // cavity tets deleted (T_deleted)
  // verification outcomes of the last check pass (diagnostics, verbose rounds):
  // [0] subsegments missing, [1] encroached by a vertex off the segment line,
  // [2] encroached by a (near-)collinear vertex, [3] subfaces missing,
  // [4] encroached by an off-plane apex, [5] encroached by a (near-)coplanar apex
  unsigned int chk[8];
  unsigned int skipr[12];            // skipped elements by kind * 4 + reason (diagnostics)
  unsigned int fail[8];              // failed-region causes (diagnostics): 0 no seed, 1 seed peeled,
                                     // 2 swallows a vertex, 3 pinched ghost boundary, 4 star check,
                                     // 5 sequential-path overflow, 6 membrane, 7 exhaustive walk scans
  int first_real;                    // no alive real tet has a lower index (hint_tet; 0 after compaction)
  unsigned long long t2st[4];        // 2D cavities (diagnostics): computed, walk steps, exhaustive scans, triangles scanned
  unsigned long long fb_slow;        // slowest fallback evaluation (diagnostics): cycles << 8 | outcome << 4 | kind
  unsigned long long vq[11];          // vertex-star queries (diagnostics): stale-start scans, tets scanned, large-arena reruns, lock spins;
                                     // walks past the deterministic cap, their randomised steps;
                                     // fallback evaluations over 10 ms: kcycles in make_cand / hull walk / seeds / region, count
};

// A tet is one 32-byte record {tv, tn} (vertices, then packed neighbour
// links): a cavity step that reads both touches one sector pair of one line.
// TetRow is one half of the interleaved array, indexed like a plain array.
struct TetRow {
  int4* p;          // record r of this half is p[2 r]
  __host__ __device__ __forceinline__ int4& operator[](size_t r) const { return p[2 * r]; }
  __host__ __device__ __forceinline__ int4* operator+(size_t r) const { return p + 2 * r; }
};

struct Dev {
  // vertices
  double* P;
  uint8_t* vorigin;
  int* vert_tet;
  int* vsid;
  int vcap;
  // tets: interleaved {tv, tn} records (tv.p is the allocation)
  TetRow tv;
  TetRow tn;
  uint8_t* alive;
  uint8_t* sub;
  uint8_t* seg;
  uint8_t* skip;
  double* ratio;
  int tcap;
  // subsegments
  int2* sg_uv;
  int* sg_sid;
  unsigned int* sg_fl;
  int sgcap;
  unsigned long long* sg_hk;
  int* sg_hv;
  unsigned int sg_hmask;
  // subfaces
  int4* sf_v;          // a<b<c, pid
  unsigned int* sf_fl;
  int sfcap;
  unsigned long long* sf_hk;
  int* sf_hv;
  unsigned int sf_hmask;
  // facet triangulations
  int4* t2v;
  uint8_t* t2alive;
  int t2cap;
  unsigned long long* he_hk;
  int* he_hv;
  unsigned int he_hmask;
  int* t2count;        // alive triangles per polygon
  // static PLC info
  int2* poly_keep;     // projection axes per polygon
  int* t2last;         // per polygon: most recently added real 2D triangle (walk start)
  uint8_t* poly_obl;   // 1: polygon not parallel to a coordinate plane (in-plane circle test in 3D)
  int* segpoly_off;    // sid -> polygons (CSR)
  int* segpoly;
  int2* sid_uv;        // original segment endpoints
  uint8_t* vapex;      // input vertex where two input segments meet at < 45 degrees (n_input entries)
  int poly_obl_hull;   // some oblique polygon lies on the convex hull (hull_guard_*, gq_cand.cuh)
  const int* poly_off; // polygon vertex cycles (CSR), resident for the inside test of non-convex ones
  const int* poly_idx;
  uint8_t* poly_convex; // 1: every 2D triangle of the polygon is inside it (no centroid test needed)
  int nsid, npoly;
  double too_close_sq, lmin2;
  Counters* ctr;
  // large arenas for vertex-star queries (around_vertex overflow path)
  int* vp_key; int* vp_val; unsigned int* vp_ep; unsigned int* vp_epoch; int* vp_stack; int* vp_lock;
  int vp_cap, vp_n;
};

__device__ __forceinline__ const double* PT(const Dev& D, int v) { return D.P + 3 * (size_t)v; }
__device__ __forceinline__ int tvk(const int4& q, int k) { return k == 0 ? q.x : (k == 1 ? q.y : (k == 2 ? q.z : q.w)); }
__device__ __forceinline__ int tnk(const Dev& D, int t, int k) {
  const int* p = reinterpret_cast<const int*>(D.tn + t);
  return p[k];
}
__device__ __forceinline__ void set_tn(const Dev& D, int t, int k, int val) { reinterpret_cast<int*>(D.tn + t)[k] = val; }
__device__ __forceinline__ void face_verts(const int4& q, int i, int* f) {
  f[0] = tvk(q, c_faces[i][0]); f[1] = tvk(q, c_faces[i][1]); f[2] = tvk(q, c_faces[i][2]);
}
__device__ __forceinline__ void sort3(int& a, int& b, int& c) {
  int t;
  if (a > b) { t = a; a = b; b = t; }
  if (b > c) { t = b; b = c; c = t; }
  if (a > b) { t = a; a = b; b = t; }
}
__device__ __forceinline__ bool has_v(const int4& q, int v) { return q.x == v || q.y == v || q.z == v || q.w == v; }

// ---------------------------------------------------------------------------
// hashing
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ unsigned long long key2(int u, int v) {   // u < v
  return ((unsigned long long)(unsigned int)u << 32) | (unsigned int)v;
}
__device__ __forceinline__ unsigned long long key3(int a, int b, int c) {  // sorted triple -> 64-bit hash
  unsigned long long h = mix64(((unsigned long long)(unsigned int)a << 32) ^ (unsigned int)b);
  h = mix64(h ^ ((unsigned long long)(unsigned int)c * 0x9E3779B97F4A7C15ull));
  return h == EMPTY_KEY ? 1ull : h;
}
__device__ __forceinline__ unsigned long long keyhe(int a, int b, int pid) {  // directed 2D edge
  unsigned long long h = mix64(((unsigned long long)(unsigned int)(a + 1) << 32) ^ (unsigned int)(b + 1));
  h = mix64(h ^ ((unsigned long long)(unsigned int)pid * 0xC2B2AE3D27D4EB4Full + 0x632BE59BD9B4E019ull));
  return h == EMPTY_KEY ? 2ull : h;
}

// insert-or-update: the slot whose key equals k gets value v
__device__ inline void ht_put(unsigned long long* hk, int* hv, unsigned int mask, unsigned long long k, int v) {
  unsigned int i = (unsigned int)mix64(k) & mask;
  for (unsigned int probe = 0; probe <= mask; ++probe) {
    unsigned long long cur = hk[i];
    if (cur == k) { hv[i] = v; return; }
    if (cur == EMPTY_KEY) {
      unsigned long long old = atomicCAS(hk + i, EMPTY_KEY, k);
      if (old == EMPTY_KEY || old == k) { hv[i] = v; return; }
    }
    i = (i + 1) & mask;
  }
  raise_err(GQ_ERR_HASH);
}
// visit every slot carrying key k (64-bit hashes may collide: callers verify)
template <class F>
__device__ inline int ht_find(const unsigned long long* hk, const int* hv, unsigned int mask, unsigned long long k, F ok) {
  unsigned int i = (unsigned int)mix64(k) & mask;
  for (unsigned int probe = 0; probe <= mask; ++probe) {
    unsigned long long cur = hk[i];
    if (cur == EMPTY_KEY) return -1;
    if (cur == k) { int v = hv[i]; if (v >= 0 && ok(v)) return v; }
    i = (i + 1) & mask;
  }
  return -1;
}

__device__ inline int seg_lookup(const Dev& D, int u, int v) {   // live subsegment record of edge (u,v)
  if (u > v) { int t = u; u = v; v = t; }
  if (u < 0) return -1;
  return ht_find(D.sg_hk, D.sg_hv, D.sg_hmask, key2(u, v), [&](int r) {
    int2 e = D.sg_uv[r];
    return e.x == u && e.y == v && (D.sg_fl[r] & RF_LIVE);
  });
}
__device__ inline int face_lookup(const Dev& D, int a, int b, int c) {   // sorted triple
  if (a < 0) return -1;
  return ht_find(D.sf_hk, D.sf_hv, D.sf_hmask, key3(a, b, c), [&](int r) {
    int4 f = D.sf_v[r];
    return f.x == a && f.y == b && f.z == c && (D.sf_fl[r] & RF_LIVE);
  });
}
__device__ inline int he_lookup(const Dev& D, int a, int b, int pid) {   // triangle holding directed edge a->b
  return ht_find(D.he_hk, D.he_hv, D.he_hmask, keyhe(a, b, pid), [&](int t) {
    if (!D.t2alive[t]) return false;
    int4 q = D.t2v[t];
    if (q.w != pid) return false;
    return (q.x == a && q.y == b) || (q.y == a && q.z == b) || (q.z == a && q.x == b);
  });
}

// ---------------------------------------------------------------------------
// small per-thread open-addressing sets in global scratch
struct ISet {      // int keys -> int value; epoch-tagged slots (O(1) clear)
  int* key;
  int* val;
  unsigned int* ep;
  unsigned int* cur; // this thread's epoch counter
  int cap;           // power of two
  __device__ void clear() { *cur += 1; }
  __device__ int find(int k) const {
    unsigned int e = *cur;
    unsigned int i = ((unsigned int)k * 2654435761u) & (cap - 1);
    for (int p = 0; p < cap; ++p) {
      if (ep[i] != e) return -1;
      if (key[i] == k) return val[i];
      i = (i + 1) & (cap - 1);
    }
    return -1;
  }
  __device__ bool put(int k, int v) {
    unsigned int e = *cur;
    unsigned int i = ((unsigned int)k * 2654435761u) & (cap - 1);
    for (int p = 0; p < cap; ++p) {
      if (ep[i] != e) { ep[i] = e; key[i] = k; val[i] = v; return true; }
      if (key[i] == k) { val[i] = v; return true; }
      i = (i + 1) & (cap - 1);
    }
    return false;
  }
};
struct LSet {      // 64-bit keys (set semantics), epoch-tagged
  unsigned long long* key;
  unsigned int* ep;
  unsigned int* cur;
  int cap;
  __device__ void clear() { *cur += 1; }
  __device__ bool has(unsigned long long k) const {
    unsigned int e = *cur;
    unsigned int i = (unsigned int)mix64(k) & (cap - 1);
    for (int p = 0; p < cap; ++p) {
      if (ep[i] != e) return false;
      if (key[i] == k) return true;
      i = (i + 1) & (cap - 1);
    }
    return false;
  }
  // returns 1 inserted, 0 present, -1 full
  __device__ int add(unsigned long long k) {
    unsigned int e = *cur;
    unsigned int i = (unsigned int)mix64(k) & (cap - 1);
    for (int p = 0; p < cap; ++p) {
      if (ep[i] != e) { ep[i] = e; key[i] = k; return 1; }
      if (key[i] == k) return 0;
      i = (i + 1) & (cap - 1);
    }
    return -1;
  }
};

// ---------------------------------------------------------------------------
// adjacency queries (mesh.py:236-282); the visited set lives in scratch
__device__ __noinline__ int first_alive_with(const Dev& D, int v) {
  int nt = D.ctr->nt;
  for (int t = 0; t < nt; ++t) if (D.alive[t] && has_v(D.tv[t], v)) return t;
  return -1;
}

// One DFS over the tets around v with the given visited set / stack.
// Returns 1 done (or stopped by f), 0 no alive tet, -1 the set or the stack
// overflowed (nothing is lost: the caller reruns with a larger arena).
template <class F>
__device__ __noinline__ int around_vertex_try(const Dev& D, int v, ISet& seen, int* stack, int cap, F& f) {
  int start = D.vert_tet[v];
  if (start < 0 || start >= D.ctr->nt || !D.alive[start] || !has_v(D.tv[start], v)) {
    start = first_alive_with(D, v);
    atomicAdd(&D.ctr->vq[0], 1ull); atomicAdd(&D.ctr->vq[1], (unsigned long long)(start < 0 ? D.ctr->nt : start + 1));
    if (start < 0) return 0;
    D.vert_tet[v] = start;   // same side effect as the reference
  }
  seen.clear();
  seen.put(start, 0);
  if (f(start)) return 1;
  int sp = 0;
  stack[sp++] = start;
  while (sp > 0) {
    int t = stack[--sp];
    int4 q = D.tv[t];
    for (int i = 0; i < 4; ++i) {
      if (tvk(q, i) == v) continue;
      int u = tnk(D, t, i) >> 2;
      if (u < 0 || !D.alive[u] || seen.find(u) >= 0) continue;
      if (!seen.put(u, 0) || sp >= cap) return -1;
      if (f(u)) return 1;
      stack[sp++] = u;
    }
  }
  return 1;
}

// Large vertex stars (a box corner joined to thousands of hull vertices, a
// vertex of a finely split small input angle): a DFS that outgrows the
// per-thread arena reruns on one of a few large arenas, taken with a lock.
// Holders never wait for anything else, so the spin always ends.
__device__ inline int vpool_acquire(const Dev& D) {
  unsigned int s0 = (unsigned int)(blockIdx.x * blockDim.x + threadIdx.x) % (unsigned int)D.vp_n;
  while (true) {
    for (int k = 0; k < D.vp_n; ++k) {
      int s = (int)((s0 + k) % (unsigned int)D.vp_n);
      if (atomicCAS(D.vp_lock + s, 0, 1) == 0) { __threadfence(); return s; }
    }
    atomicAdd(&D.ctr->vq[3], 1ull);
    __nanosleep(256);
  }
}
__device__ inline void vpool_release(const Dev& D, int s) { __threadfence(); atomicExch(D.vp_lock + s, 0); }

// visit tets around vertex v; f(t) returns true to stop early.  Returns
// false when v has no alive tet.  When the per-thread arena overflows, the
// walk restarts on a large arena after reset() (f may see a tet twice).
template <class F, class R>
__device__ inline bool around_vertex(const Dev& D, int v, ISet& seen, int* stack, int cap, F f, R reset) {
  int r = around_vertex_try(D, v, seen, stack, cap, f);
  if (r >= 0) return r > 0;
  reset();
  atomicAdd(&D.ctr->vq[2], 1ull);
  int s = vpool_acquire(D);
  ISet big;
  size_t o = (size_t)s * D.vp_cap;
  big.key = D.vp_key + o; big.val = D.vp_val + o; big.ep = D.vp_ep + o; big.cur = D.vp_epoch + s; big.cap = D.vp_cap;
  r = around_vertex_try(D, v, big, D.vp_stack + o, D.vp_cap, f);
  vpool_release(D, s);
  if (r < 0) raise_err(GQ_ERR_CAP);
  return r > 0;
}
template <class F>
__device__ inline bool around_vertex(const Dev& D, int v, ISet& seen, int* stack, int cap, F f) {
  return around_vertex(D, v, seen, stack, cap, f, [] {});
}
// Visit the tets of edge (u,v) (f(t) may stop early): the DFS around u on the
// per-thread arena; when u's star outgrows it (a box corner is joined to
// thousands of hull vertices), the star of v, which holds the same edge tets,
// on the per-thread arena; only when both overflow, u on a large arena.  The
// visited set is the same either way; u's stale vert_tet entry is repaired by
// the first attempt exactly as before.
template <class F, class R>
__device__ inline bool around_edge(const Dev& D, int u, int v, ISet& seen, int* stack, int cap, F f, R reset) {
  auto fu = [&](int t) { return has_v(D.tv[t], v) ? f(t) : false; };
  int r = around_vertex_try(D, u, seen, stack, cap, fu);
  if (r >= 0) return r > 0;
  reset();
  auto fv = [&](int t) { return has_v(D.tv[t], u) ? f(t) : false; };
  r = around_vertex_try(D, v, seen, stack, cap, fv);
  if (r >= 0) return r > 0;
  reset();
  return around_vertex(D, u, seen, stack, cap, fu, reset);
}
__device__ inline bool edge_exists(const Dev& D, int u, int v, ISet& seen, int* stack, int cap) {
  bool found = false;
  around_edge(D, u, v, seen, stack, cap, [&](int) { found = true; return true; }, [] {});
  return found;
}
// (t,i) of an alive tet with face {a,b,c} (sorted), or t=-1
__device__ inline int find_face(const Dev& D, int a, int b, int c, ISet& seen, int* stack, int cap) {
  int res = -1;
  around_vertex(D, a, seen, stack, cap, [&](int t) {
    int4 q = D.tv[t];
    if (!has_v(q, b) || !has_v(q, c)) return false;
    for (int i = 0; i < 4; ++i) {
      int f[3]; face_verts(q, i, f); sort3(f[0], f[1], f[2]);
      if (f[0] == a && f[1] == b && f[2] == c) { res = 4 * t + i; return true; }
    }
    return false;
  });
  return res;
}

// ---------------------------------------------------------------------------
// walks (mesh.py:307-371)
// mesh.py:307-320: the hint, else the lowest-index alive real tet.  Tet slots
// only die or are appended between compactions, so that index never
// decreases: the scan starts at the last one found (D.ctr->first_real) and
// returns exactly what a scan from slot 0 would.
__device__ __noinline__ int hint_tet(const Dev& D, int hint) {
  int nt = D.ctr->nt;
  if (hint >= 0 && hint < nt && D.alive[hint] && D.tv[hint].w != GHOST) return hint;
  for (int t = max(D.ctr->first_real, 0); t < nt; ++t)
    if (D.alive[t] && D.tv[t].w != GHOST) { atomicMax(&D.ctr->first_real, t); return t; }
  raise_err(GQ_ERR_WALK);
  return 0;
}
__device__ inline int walk_cap(const Dev& D, int extra) {
  double nt = D.ctr->nt > 1 ? (double)D.ctr->nt : 1.0;
  return (int)(10.0 * pow(nt, 1.0 / 3.0)) + extra;
}
// closed containment of p in real tet t (every face orient3d <= 0)
__device__ inline bool contains_closed(const Dev& D, int t, const double* p) {
  int4 q = D.tv[t];
  for (int i = 0; i < 4; ++i) {
    int f[3]; face_verts(q, i, f);
    if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) > 0) return false;
  }
  return true;
}
// The exhaustive scan below returns the lowest-index real tet containing p
// (else the lowest-index ghost whose hull face sees p).  Those tets form a
// face-connected set around the tet a walk ends in (the tets sharing the
// face / edge / vertex p lies on; the visible part of the convex hull), so a
// bounded search from there gives the same answer; -1 when the set is larger
// than the search's arena.
__device__ __noinline__ int lowest_equivalent(const Dev& D, const double* p, int t0) {
  const int CAP = 96;
  int found[CAP];
  int n = 0, head = 0;
  bool ghost = D.tv[t0].w == GHOST;
  found[n++] = t0;
  int best = t0;
  while (head < n) {
    int cur = found[head++];
    int4 q = D.tv[cur];
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, cur, i) >> 2;
      if (u < 0 || !D.alive[u]) continue;
      int4 qu = D.tv[u];
      bool member;
      if (ghost) {
        if (qu.w != GHOST) continue;
        member = orient3d(PT(D, qu.x), PT(D, qu.y), PT(D, qu.z), p) > 0;
      } else {
        if (qu.w == GHOST) continue;
        int f[3]; face_verts(q, i, f);
        if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) != 0) continue;   // p not on the shared face
        member = contains_closed(D, u, p);
      }
      if (!member) continue;
      bool seen = false;
      for (int k = 0; k < n && !seen; ++k) seen = found[k] == u;
      if (seen) continue;
      if (n >= CAP) return -1;
      found[n++] = u;
      if (u < best) best = u;
    }
  }
  return best;
}
__device__ __noinline__ int walk(const Dev& D, const double* p, int hint) {
  int t = hint_tet(D, hint);
  int max_steps = walk_cap(D, 32);
  int step = 0, prev = -1;
  while (step < max_steps) {
    step += 1;
    int4 q = D.tv[t];
    if (q.w == GHOST) return t;
    bool moved = false;
    for (int k = 0; k < 4; ++k) {
      int i = (k + step) & 3;
      int u = tnk(D, t, i) >> 2;
      if (u == prev) continue;
      int f[3]; face_verts(q, i, f);
      if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) > 0) { prev = t; t = u; moved = true; break; }
    }
    if (!moved) return t;
  }
  {
    // The deterministic walk cycled (it can on a constrained mesh).  Where
    // the reference scans every tet (mesh.py:362-371), first finish with a
    // randomised remembering walk, which leaves any cycle, and resolve the
    // scan's tie rule locally (lowest_equivalent): same tet, no O(nt) pass.
    unsigned long long r = 0x9E3779B97F4A7C15ull ^ (unsigned long long)t;
    prev = -1;
    atomicAdd(&D.ctr->vq[4], 1ull);
    int s2 = 0;
    for (; s2 < 16 * max_steps; ++s2) {
      int4 q = D.tv[t];
      if (q.w == GHOST) break;
      if ((s2 & 255) == 255) atomicAdd(&D.ctr->vq[5], 256ull);
      r = r * 6364136223846793005ull + 1442695040888963407ull;
      int off = (int)(r >> 62);
      bool moved = false;
      for (int k = 0; k < 4; ++k) {
        int i = (k + off) & 3;
        int u = tnk(D, t, i) >> 2;
        if (u == prev) continue;
        int f[3]; face_verts(q, i, f);
        if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) > 0) { prev = t; t = u; moved = true; break; }
      }
      if (!moved) {
        int b = lowest_equivalent(D, p, t);
        if (b >= 0) return b;
        break;
      }
    }
    if (D.tv[t].w == GHOST) {
      int4 q = D.tv[t];
      if (orient3d(PT(D, q.x), PT(D, q.y), PT(D, q.z), p) > 0) {
        // outside the hull: the reference returns the lowest ghost seeing p, but only when
        // no real tet contains p -- true here, since the walk left the hull through a visible face
        int b = lowest_equivalent(D, p, t);
        if (b >= 0) return b;
      }
    }
  }
  int nt = D.ctr->nt;
  atomicAdd(&D.ctr->fail[7], 1u);
  for (int s = 0; s < nt; ++s) {
    if (!D.alive[s] || D.tv[s].w == GHOST) continue;
    int4 q = D.tv[s];
    bool in = true;
    for (int i = 0; i < 4 && in; ++i) {
      int f[3]; face_verts(q, i, f);
      if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) > 0) in = false;
    }
    if (in) return s;
  }
  for (int s = 0; s < nt; ++s) {
    if (D.alive[s] && D.tv[s].w == GHOST) {
      int4 q = D.tv[s];
      if (orient3d(PT(D, q.x), PT(D, q.y), PT(D, q.z), p) > 0) return s;
    }
  }
  raise_err(GQ_ERR_WALK);
  return -1;
}

// ---------------------------------------------------------------------------
// allowed_cross as a predicate: a face is crossable iff it is a live subface
// whose polygon is one of the candidate's polygons (refine.py:359-370)
struct Allow {
  int pid[4];
  int n;
  const int* many;   // n > 4: the segment's polygon list (D.segpoly), pid[] unused
  __device__ bool any() const { return n > 0; }
  __device__ int at(int k) const { return n <= 4 ? pid[k] : many[k]; }
};
__device__ __noinline__ bool allowed_face(const Dev& D, const Allow& A, int a, int b, int c) {
  if (A.n == 0) return false;
  sort3(a, b, c);
  int r = face_lookup(D, a, b, c);
  if (r < 0) return false;
  int pid = D.sf_v[r].w;
  for (int k = 0; k < A.n; ++k) if (A.at(k) == pid) return true;
  return false;
}
__device__ inline bool blocked(const Dev& D, const Allow& A, int t, int i) {
  if (!(D.sub[t] & (1 << i))) return false;
  if (A.n == 0) return true;
  int f[3]; face_verts(D.tv[t], i, f);
  return !allowed_face(D, A, f[0], f[1], f[2]);
}
// mesh.py:395-414
__device__ __noinline__ bool in_region(const Dev& D, int t, const double* p, const Allow& A) {
  int4 q = D.tv[t];
  if (q.w == GHOST) {
    const double *a = PT(D, q.x), *b = PT(D, q.y), *c = PT(D, q.z);
    int s = orient3d(a, b, c, p);
    if (s > 0) return true;
    if (s == 0) return incircle3d(a, b, c, p) > 0;
    if (A.n > 0 && allowed_face(D, A, q.x, q.y, q.z)) return incircle3d(a, b, c, p) > 0;
    return false;
  }
  return insphere(PT(D, q.x), PT(D, q.y), PT(D, q.z), PT(D, q.w), p) > 0;
}

// ---------------------------------------------------------------------------
// Delaunay region (mesh.py:450-521, decisions of _kernels.py:392-635)
enum RegionStatus { RS_OK = 0, RS_CNSS = 1, RS_MEMBRANE = 2, RS_OVERFLOW = 3, RS_TOOCLOSE = 4, RS_BADSTAR = 5,
                    RS_SHRUNK = 6 /* internal: seed peeled, retry with the next seed */ };

// Star validation before anything is written.  The peel makes every real
// boundary face strictly visible from p, so a cavity of real tets always
// stars; faces through the ghost vertex are not tested by the peel, and a
// point that rounds to just outside a curved hull can leave a pinched
// boundary.  The reference notices only while starring (star_kernel's
// unmatched-face status, _kernels.py:696,720 -> CavityNotStarShaped,
// mesh.py:769-770).  Here the cavity is rejected up front (RS_BADSTAR -> a
// failed candidate, and the sequential fallback skips it with reason
// cavity_not_star_shaped, refine.py:785-799) when some boundary-face edge
// (ghost vertex included) lies on other than exactly two boundary faces.
// Faces [r, r+stride, ...) are checked by the caller's lane r.
__device__ inline bool bf_has_ghost_part(const Dev& D, const int* bf, int nbf, int r, int stride) {
  for (int k = r; k < nbf; k += stride) {
    int f[3]; face_verts(D.tv[bf[k] >> 2], bf[k] & 3, f);
    if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) return true;
  }
  return false;
}
__device__ inline bool bf_open_part(const Dev& D, const int* bf, int nbf, int r, int stride) {
  for (int k = r; k < nbf; k += stride) {
    int f[3]; face_verts(D.tv[bf[k] >> 2], bf[k] & 3, f);
    for (int e = 0; e < 3; ++e) {
      int x = f[e], y = f[(e + 1) % 3];
      int cnt = 0;
      for (int j = 0; j < nbf && cnt <= 2; ++j) {
        int g[3]; face_verts(D.tv[bf[j] >> 2], bf[j] & 3, g);
        cnt += (g[0] == x || g[1] == x || g[2] == x) && (g[0] == y || g[1] == y || g[2] == y);
      }
      if (cnt != 2) return true;
    }
  }
  return false;
}

// Linear-time forms of bf_open_part (same answer): every boundary-face edge is
// counted in a hash instead of against every other face.
//  - one thread: two tagged keys per edge in the thread's 64-bit set (the set
//    keeps its other keys; a full set falls back to the quadratic count);
//  - a block: the count packed into the key of a raw table on the block's
//    64-bit arena (cleared first; the set's epoch is bumped afterwards so its
//    own users see it empty).  Call with every thread of the block.
__device__ __forceinline__ unsigned long long bf_edge_key(int a, int b) {
  int x = a + 1, y = b + 1;   // ghost (-1) -> 0
  if (x > y) { int t = x; x = y; y = t; }
  return ((unsigned long long)(unsigned)x << 30) | (unsigned long long)(unsigned)y;
}
__device__ inline bool bf_open_seq(const Dev& D, const int* bf, int nbf, LSet& F) {
  const unsigned long long T1 = 8ull << 60, T2 = 9ull << 60;
  for (int k = 0; k < nbf; ++k) {
    int f[3]; face_verts(D.tv[bf[k] >> 2], bf[k] & 3, f);
    for (int e = 0; e < 3; ++e) {
      unsigned long long E = bf_edge_key(f[e], f[(e + 1) % 3]);
      int a = F.add(T1 | E);
      if (a < 0) return bf_open_part(D, bf, nbf, 0, 1);
      if (a == 1) continue;
      a = F.add(T2 | E);
      if (a < 0) return bf_open_part(D, bf, nbf, 0, 1);
      if (a == 0) return true;            // a third face on this edge
    }
  }
  for (int k = 0; k < nbf; ++k) {
    int f[3]; face_verts(D.tv[bf[k] >> 2], bf[k] & 3, f);
    for (int e = 0; e < 3; ++e)
      if (!F.has(T2 | bf_edge_key(f[e], f[(e + 1) % 3]))) return true;   // a single face on this edge
  }
  return false;
}
__device__ inline bool bf_open_block(const Dev& D, const int* bf, int nbf, LSet& F, int nthreads) {
  const int tid = threadIdx.x;
  if ((long long)F.cap < 4LL * nbf) return __syncthreads_or(bf_open_part(D, bf, nbf, tid, nthreads));
  volatile unsigned long long* K = F.key;
  for (int i = tid; i < F.cap; i += nthreads) K[i] = 0ull;
  __syncthreads();
  for (int k = tid; k < nbf; k += nthreads) {
    int f[3]; face_verts(D.tv[bf[k] >> 2], bf[k] & 3, f);
    for (int e = 0; e < 3; ++e) {
      unsigned long long E = bf_edge_key(f[e], f[(e + 1) % 3]) << 2;   // low 2 bits: count (saturating at 3)
      unsigned int i = (unsigned int)mix64(E) & (unsigned int)(F.cap - 1);
      while (true) {
        unsigned long long cur = K[i];
        if (cur == 0ull) {
          cur = atomicCAS(&F.key[i], 0ull, E | 1ull);
          if (cur == 0ull) break;
        }
        if ((cur >> 2) == (E >> 2)) {
          while ((cur & 3ull) != 3ull) {
            unsigned long long old = atomicCAS(&F.key[i], cur, cur + 1ull);
            if (old == cur) break;
            cur = old;
          }
          break;
        }
        i = (i + 1) & (unsigned int)(F.cap - 1);
      }
    }
  }
  __syncthreads();
  bool bad = false;
  for (int i = tid; i < F.cap && !bad; i += nthreads) {
    unsigned long long v = K[i];
    bad = v != 0ull && (v & 3ull) != 2ull;
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) F.clear();
  __syncthreads();
  return bad;
}

struct Scratch {     // per-thread scratch views
  ISet tset;         // tet -> list index
  LSet fset;         // tagged keys: vertices, edges, faces
  int* list;         // cavity tets (grown order)
  int* stack;
  uint8_t* in;
  uint8_t* comp;
  int cap;           // max tets
  // fallback scan (k_fb_scan): the evaluation of list entry `me` is abandoned
  // once an earlier entry has broken the wave (*cancel < me); null elsewhere
  const int* cancel;
  int me;
};

struct RegionOut {   // output slab views (capacities given)
  int* tets; int* bf; int* cr; int* crf; int* bsub; int* bseg; int* eseg;
  int ctet, cbf, ccon;
  int ntet, nbf, ncr, nbsub, nbseg, neseg;
  double mind;
  int memb;          // membrane face (4t+i) when RS_MEMBRANE
  int seed;
  // redirect probe (refine.py:595-662 via the grown cavity):
  // 0 off, 1 subsegments, 2 subsegments + subfaces
  int probe;
  int* rseg; int* rface; int crd;
  int nrseg, nrface;
};

// grow only (used to find the constraints a splitting point may encroach)
// then peel, component and finish.  Returns a RegionStatus.
__device__ __noinline__ int region_compute(const Dev& D, const double* p, const int* seeds, int nseeds, const Allow& A,
                                     Scratch& S, RegionOut& O, bool walk_on_miss = true) {
  int seed = -1;
  int cands[8];
  int nc = nseeds < 8 ? nseeds : 8;
  for (int k = 0; k < nc; ++k) cands[k] = seeds[k];
  bool walked = false;
  while (true) {
    seed = -1;
    for (int k = 0; k < nc; ++k) {
      int t = cands[k];
      if (t < 0 || !D.alive[t]) continue;
      if (in_region(D, t, p, A)) { seed = t; break; }
    }
    if (seed >= 0) break;
    if (walked || !walk_on_miss) return RS_CNSS;
    walked = true;
    int t = walk(D, p, nc > 0 ? cands[0] : -1);
    if (t < 0) return RS_CNSS;
    cands[0] = t; nc = 1;
  }
  O.seed = seed;
  // grow (DFS)
  S.tset.clear();
  int n = 0;
  S.list[n] = seed; S.in[n] = 1; S.tset.put(seed, n); ++n;
  int sp = 0;
  S.stack[sp++] = seed;
  while (sp > 0) {
    if (S.cancel && (sp & 15) == 0 && *(const volatile int*)S.cancel < S.me) return RS_CNSS;   // result unused
    int t = S.stack[--sp];
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, t, i) >> 2;
      if (u < 0 || !D.alive[u] || S.tset.find(u) >= 0) continue;
      if (blocked(D, A, t, i)) continue;
      if (in_region(D, u, p, A)) {
        if (n >= S.cap) return RS_OVERFLOW;
        S.list[n] = u; S.in[n] = 1;
        if (!S.tset.put(u, n)) return RS_OVERFLOW;
        ++n;
        S.stack[sp++] = u;
      }
    }
  }
  if (O.probe) {
    // constraints touched by the grown cavity whose open ball holds p
    S.fset.clear();
    O.nrseg = 0; O.nrface = 0;
    for (int k = 0; k < n; ++k) {
      int t = S.list[k];
      int4 q = D.tv[t];
      int em = D.seg[t];
      for (int i = 0; em && i < 6; ++i) {
        if (!(em & (1 << i))) continue;
        int x = tvk(q, c_edges[i][0]), y = tvk(q, c_edges[i][1]);
        if (x > y) { int tt = x; x = y; y = tt; }
        int ins = S.fset.add((5ull << 60) | ((unsigned long long)x << 30) | (unsigned long long)y);
        if (ins < 0) return RS_OVERFLOW;
        if (ins == 0) continue;
        int rec = seg_lookup(D, x, y);
        if (rec < 0 || (D.sg_fl[rec] & RF_SKIP)) continue;
        if (encroaches_segment(PT(D, x), PT(D, y), p)) {
          if (O.nrseg >= O.crd) { raise_err(GQ_ERR_CAP); return RS_OVERFLOW; }
          O.rseg[O.nrseg++] = rec;
        }
      }
      int sm = O.probe == 2 ? D.sub[t] : 0;
      for (int i = 0; sm && i < 4; ++i) {
        if (!(sm & (1 << i))) continue;
        int f[3]; face_verts(q, i, f); sort3(f[0], f[1], f[2]);
        int ins = S.fset.add((6ull << 60) | (key3(f[0], f[1], f[2]) & ((1ull << 60) - 1)));
        if (ins < 0) return RS_OVERFLOW;
        if (ins == 0) continue;
        int rec = face_lookup(D, f[0], f[1], f[2]);
        if (rec < 0 || (D.sf_fl[rec] & RF_SKIP)) continue;
        if (encroaches_face(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p)) {
          if (O.nrface >= O.crd) { raise_err(GQ_ERR_CAP); return RS_OVERFLOW; }
          O.rface[O.nrface++] = rec;
        }
      }
    }
  }
  // peel to the largest star-shaped subset, keep the seed component, repeat
  int seedk = 0;
  while (true) {
    // worklist form of the confluent peel: only neighbours of a removed tet
    // can change state, so each tet is re-examined O(1) times.  comp[] marks
    // queued entries; stack holds the queue.
    int qn = 0;
    for (int k = 0; k < n; ++k) if (S.in[k]) { S.stack[qn++] = k; S.comp[k] = 1; } else S.comp[k] = 0;
    while (qn > 0) {
      int k = S.stack[--qn];
      S.comp[k] = 0;
      if (!S.in[k]) continue;
      int t = S.list[k];
      int4 q = D.tv[t];
      bool rm = false;
      for (int i = 0; i < 4 && !rm; ++i) {
        int u = tnk(D, t, i) >> 2;
        bool blk = blocked(D, A, t, i);
        int ku = S.tset.find(u);
        bool uin = ku >= 0 && S.in[ku];
        if (uin && !blk) continue;
        int f[3]; face_verts(q, i, f);
        if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) continue;
        if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) >= 0) rm = true;
      }
      if (!rm) continue;
      S.in[k] = 0;
      for (int i = 0; i < 4; ++i) {
        int ku = S.tset.find(tnk(D, t, i) >> 2);
        if (ku >= 0 && S.in[ku] && !S.comp[ku]) { S.comp[ku] = 1; S.stack[qn++] = ku; }
      }
    }
    if (!S.in[seedk]) return RS_CNSS;   // seed shrunk away
    int live = 0;
    for (int k = 0; k < n; ++k) { live += S.in[k]; S.comp[k] = 0; }
    int ncomp = 1;
    S.comp[seedk] = 1;
    sp = 0;
    S.stack[sp++] = seed;
    while (sp > 0) {
      int t = S.stack[--sp];
      for (int i = 0; i < 4; ++i) {
        int u = tnk(D, t, i) >> 2;
        int ku = S.tset.find(u);
        if (ku < 0 || !S.in[ku] || S.comp[ku]) continue;
        if (blocked(D, A, t, i)) continue;
        S.comp[ku] = 1; ++ncomp;
        S.stack[sp++] = u;
      }
    }
    if (ncomp == live) break;
    for (int k = 0; k < n; ++k) S.in[k] = S.comp[k];
  }
  // finish: cavity tets sorted by id
  int m = 0;
  for (int k = 0; k < n; ++k) if (S.in[k]) S.stack[m++] = S.list[k];
  if (m <= 48) {
    for (int a = 1; a < m; ++a) {         // insertion sort (typical regions are small)
      int x = S.stack[a], b = a - 1;
      while (b >= 0 && S.stack[b] > x) { S.stack[b + 1] = S.stack[b]; --b; }
      S.stack[b + 1] = x;
    }
  } else {
    int* h = S.stack;                      // heap sort for big cavities
    auto sift = [&](int root, int end) {
      while (2 * root + 1 < end) {
        int ch = 2 * root + 1;
        if (ch + 1 < end && h[ch] < h[ch + 1]) ++ch;
        if (h[root] >= h[ch]) return;
        int t = h[root]; h[root] = h[ch]; h[ch] = t;
        root = ch;
      }
    };
    for (int a = m / 2 - 1; a >= 0; --a) sift(a, m);
    for (int e = m - 1; e > 0; --e) { int t = h[0]; h[0] = h[e]; h[e] = t; sift(0, e); }
  }
  if (m > O.ctet) return RS_OVERFLOW;
  O.ntet = m; O.nbf = 0; O.ncr = 0; O.nbsub = 0; O.nbseg = 0; O.neseg = 0;
  S.fset.clear();
  const unsigned long long TV = 1ull << 60, TE = 2ull << 60, TSF = 3ull << 60, TSG = 4ull << 60;
  // boundary-edge "first tet index" must be known for the subsegment rule:
  // a subsegment is boundary iff its edge is on a boundary face of a tet
  // visited no later than the tet where the subsegment is first met
  for (int a = 0; a < m; ++a) {
    int t = S.stack[a];
    O.tets[a] = t;
    int4 q = D.tv[t];
    for (int i = 0; i < 4; ++i) {
      int u = tnk(D, t, i) >> 2;
      bool blk = blocked(D, A, t, i);
      int ku = S.tset.find(u);
      bool uin = ku >= 0 && S.in[ku];
      if (uin && !blk) continue;
      if (uin && blk) { O.memb = 4 * t + i; return RS_MEMBRANE; }
      if (O.nbf >= O.cbf) return RS_OVERFLOW;
      O.bf[O.nbf++] = 4 * t + i;
      int f[3]; face_verts(q, i, f);
      for (int k = 0; k < 3; ++k) if (f[k] != GHOST && S.fset.add(TV | (unsigned int)f[k]) < 0) return RS_OVERFLOW;
      for (int k = 0; k < 3; ++k) {
        int x = f[k], y = f[(k + 1) % 3];
        if (x == GHOST || y == GHOST) continue;
        if (x > y) { int tt = x; x = y; y = tt; }
        if (S.fset.add(TE | ((unsigned long long)x << 30) | (unsigned long long)y) < 0) return RS_OVERFLOW;
      }
    }
    int sm = D.sub[t];
    if (sm) {
      for (int i = 0; i < 4; ++i) {
        if (!(sm & (1 << i))) continue;
        int f[3]; face_verts(q, i, f);
        int a0 = f[0], b0 = f[1], c0 = f[2];
        sort3(a0, b0, c0);
        unsigned long long fk = TSF | (key3(a0, b0, c0) & ((1ull << 60) - 1));
        int ins = S.fset.add(fk);
        if (ins < 0) return RS_OVERFLOW;
        if (ins == 0) continue;
        int u = tnk(D, t, i) >> 2;
        int ku = S.tset.find(u);
        bool uin = ku >= 0 && S.in[ku];
        int rec = face_lookup(D, a0, b0, c0);
        bool crossed = uin && rec >= 0 && A.n > 0 && allowed_face(D, A, a0, b0, c0);
        if (crossed) {
          if (O.ncr >= O.ccon) return RS_OVERFLOW;
          O.cr[O.ncr] = rec;
          O.crf[O.ncr] = min(4 * t + i, tnk(D, t, i));
          O.ncr++;
        } else {
          if (O.nbsub >= O.ccon) return RS_OVERFLOW;
          O.bsub[O.nbsub++] = rec;
        }
      }
    }
    int em = D.seg[t];
    if (em) {
      for (int i = 0; i < 6; ++i) {
        if (!(em & (1 << i))) continue;
        int x = tvk(q, c_edges[i][0]), y = tvk(q, c_edges[i][1]);
        if (x > y) { int tt = x; x = y; y = tt; }
        int ins = S.fset.add(TSG | ((unsigned long long)x << 30) | (unsigned long long)y);
        if (ins < 0) return RS_OVERFLOW;
        if (ins == 0) continue;
        int rec = seg_lookup(D, x, y);
        bool bound = S.fset.has(TE | ((unsigned long long)x << 30) | (unsigned long long)y);
        if (O.nbseg + O.neseg >= O.ccon) return RS_OVERFLOW;
        if (bound) O.bseg[O.nbseg++] = rec; else O.eseg[O.neseg++] = rec;
      }
    }
  }
  // (sequential path: every cavity is checked, see k_star_check for why the peel is not enough)
  if (bf_open_seq(D, O.bf, O.nbf, S.fset)) return RS_BADSTAR;
  double mind = __longlong_as_double(0x7ff0000000000000ll);
  for (int a = 0; a < O.nbf; ++a) {
    int t = O.bf[a] >> 2, i = O.bf[a] & 3;
    int f[3]; face_verts(D.tv[t], i, f);
    for (int k = 0; k < 3; ++k) {
      if (f[k] == GHOST) continue;
      const double* qv = PT(D, f[k]);
      double d = (qv[0] - p[0]) * (qv[0] - p[0]) + (qv[1] - p[1]) * (qv[1] - p[1]) + (qv[2] - p[2]) * (qv[2] - p[2]);
      if (d < mind) mind = d;
    }
  }
  O.mind = mind;
  for (int a = 0; a < m; ++a) {
    int4 q = D.tv[O.tets[a]];
    for (int k = 0; k < 4; ++k) {
      int v = tvk(q, k);
      if (v != GHOST && !S.fset.has(TV | (unsigned int)v)) return RS_CNSS;   // swallows a vertex
    }
  }
  return RS_OK;
}

// ---------------------------------------------------------------------------
// Bowyer-Watson star of one cavity (mesh.py:697-771, _kernels.py:641-807).
// New tets nt0..nt0+nbf-1 are created in boundary-face order.  Masks are
// taken from the (already updated) constraint tables.
__device__ __noinline__ void star_ratio(const Dev& D, int t) {
  int4 q = D.tv[t];
  if (q.w == GHOST) { D.ratio[t] = -1.0; return; }
  const double *A = PT(D, q.x), *Bp = PT(D, q.y), *C = PT(D, q.z), *Dd = PT(D, q.w);
  double ax = A[0], ay = A[1], az = A[2];
  double ux = Bp[0] - ax, uy = Bp[1] - ay, uz = Bp[2] - az;
  double vx = C[0] - ax, vy = C[1] - ay, vz = C[2] - az;
  double wx = Dd[0] - ax, wy = Dd[1] - ay, wz = Dd[2] - az;
  double vwx = vy * wz - vz * wy, vwy = vz * wx - vx * wz, vwz = vx * wy - vy * wx;
  double denom = 2.0 * (ux * vwx + uy * vwy + uz * vwz);
  if (denom == 0.0 || !isfinite(denom)) {
    // mesh.py:213-232 exact fallback
    Sphere s;
    if (circumsphere_tet(A, Bp, C, Dd, s) != 0) { D.ratio[t] = __longlong_as_double(0x7ff0000000000000ll); return; }
    double sh = dist2(A, Bp);
    double d;
    d = dist2(A, C); if (d < sh) sh = d;
    d = dist2(A, Dd); if (d < sh) sh = d;
    d = dist2(Bp, C); if (d < sh) sh = d;
    d = dist2(Bp, Dd); if (d < sh) sh = d;
    d = dist2(C, Dd); if (d < sh) sh = d;
    D.ratio[t] = sqrt(s.r2 / sh);
    return;
  }
  double lu = ux * ux + uy * uy + uz * uz;
  double lv = vx * vx + vy * vy + vz * vz;
  double lw = wx * wx + wy * wy + wz * wz;
  double wux = wy * uz - wz * uy, wuy = wz * ux - wx * uz, wuz = wx * uy - wy * ux;
  double uvx = uy * vz - uz * vy, uvy = uz * vx - ux * vz, uvz = ux * vy - uy * vx;
  double ox = (lu * vwx + lv * wux + lw * uvx) / denom;
  double oy = (lu * vwy + lv * wuy + lw * uvy) / denom;
  double oz = (lu * vwz + lv * wuz + lw * uvz) / denom;
  double r2 = ox * ox + oy * oy + oz * oz;
  double sh = lu;
  if (lv < sh) sh = lv;
  if (lw < sh) sh = lw;
  double d2 = dist2(C, Bp); if (d2 < sh) sh = d2;
  d2 = dist2(Dd, Bp); if (d2 < sh) sh = d2;
  d2 = dist2(Dd, C); if (d2 < sh) sh = d2;
  D.ratio[t] = sqrt(r2 / sh);
}

__device__ __noinline__ void refresh_masks(const Dev& D, int t) {   // mesh.py:827-840
  int4 q = D.tv[t];
  int sm = 0;
  for (int i = 0; i < 4; ++i) {
    int f[3]; face_verts(q, i, f);
    if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) continue;
    sort3(f[0], f[1], f[2]);
    if (face_lookup(D, f[0], f[1], f[2]) >= 0) sm |= 1 << i;
  }
  D.sub[t] = (uint8_t)sm;
  int em = 0;
  for (int i = 0; i < 6; ++i) {
    int a = tvk(q, c_edges[i][0]), b = tvk(q, c_edges[i][1]);
    if (a != GHOST && b != GHOST && seg_lookup(D, a, b) >= 0) em |= 1 << i;
  }
  D.seg[t] = (uint8_t)em;
}

// creates the star; returns false on a wiring failure.  When max_vt is true
// vertex->tet links use atomicMax (concurrent stars in one round: the
// sequential reference leaves each vertex pointing at its highest new tet).
__device__ __noinline__ bool star_insert(const Dev& D, int vid, const int* bf, int nbf, int nt0, bool max_vt) {
  for (int k = 0; k < nbf; ++k) {
    int t = bf[k] >> 2, i = bf[k] & 3;
    int packed = tnk(D, t, i);
    int u = packed >> 2, j = packed & 3;
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
    D.tn[nt] = make_int4(-1, -1, -1, -1);
    D.alive[nt] = 1; D.sub[nt] = 0; D.seg[nt] = 0; D.skip[nt] = 0;
    for (int m = 0; m < 4; ++m) {
      int v = tvk(q, m);
      if (v == GHOST || v == vid) continue;
      if (max_vt) atomicMax(D.vert_tet + v, nt); else D.vert_tet[v] = nt;
    }
    int a0 = f[0], b0 = f[1], c0 = f[2];
    sort3(a0, b0, c0);
    int outer = -1;
    for (int m = 0; m < 4; ++m) {
      int g[3]; face_verts(q, m, g); sort3(g[0], g[1], g[2]);
      if (g[0] == a0 && g[1] == b0 && g[2] == c0) { outer = m; break; }
    }
    if (outer < 0) { raise_err(GQ_ERR_STAR); return false; }
    set_tn(D, nt, outer, 4 * u + j);
    set_tn(D, u, j, 4 * nt + outer);
  }
  // inner wiring: faces through vid; match by sorted vertex triple
  for (int k = 0; k < nbf; ++k) {
    int nt = nt0 + k;
    int4 q = D.tv[nt];
    for (int i = 0; i < 4; ++i) {
      if (tnk(D, nt, i) >= 0) continue;
      int f[3]; face_verts(q, i, f); sort3(f[0], f[1], f[2]);
      bool done = false;
      for (int k2 = k + 1; k2 < nbf && !done; ++k2) {
        int nt2 = nt0 + k2;
        int4 q2 = D.tv[nt2];
        for (int i2 = 0; i2 < 4; ++i2) {
          if (tnk(D, nt2, i2) >= 0) continue;
          int g[3]; face_verts(q2, i2, g); sort3(g[0], g[1], g[2]);
          if (g[0] == f[0] && g[1] == f[1] && g[2] == f[2]) {
            set_tn(D, nt, i, 4 * nt2 + i2);
            set_tn(D, nt2, i2, 4 * nt + i);
            done = true;
            break;
          }
        }
      }
      if (!done) { raise_err(GQ_ERR_STAR); return false; }
    }
  }
  for (int k = 0; k < nbf; ++k) {
    int nt = nt0 + k;
    refresh_masks(D, nt);
    star_ratio(D, nt);
  }
  D.vert_tet[vid] = nt0;
  return true;
}

// ---------------------------------------------------------------------------
// facet 2D triangulations (facets.py:30-236)
__device__ __forceinline__ void proj2(const Dev& D, int pid, const double* p3, double* p2) {
  int2 kp = D.poly_keep[pid];
  p2[0] = p3[kp.x]; p2[1] = p3[kp.y];
}
struct Tri2Ctx {
  const Dev* D;
  int pid;
  int vid;           // vertex being inserted (its 2D position is p)
  double p[2];
  int follow3d;      // oblique polygon: the 2D cavity is the 3D cavity's crossed subfaces (see tri2_cavity)
  __device__ void pos(int v, double* out) const {
    if (v == vid) { out[0] = p[0]; out[1] = p[1]; return; }
    proj2(*D, pid, PT(*D, v), out);
  }
};
// facets.py:92-105
__device__ inline bool tri_in_region(const Tri2Ctx& C, int tid) {
  int4 t = C.D->t2v[tid];
  double pa[2], pb[2];
  if (t.z == GHOST) {
    C.pos(t.x, pa); C.pos(t.y, pb);
    int s = orient2d(pa, pb, C.p);
    if (s != 0) return s > 0;
    return between2d_exact(pa, pb, C.p);
  }
  if (C.D->poly_obl[C.pid]) {
    // Oblique polygon: the projection to the kept axes is affine but not a
    // similarity, so the projected incircle test would build a triangulation
    // that disagrees with the 3D mesh's subfaces (whose Delaunay property is
    // the equatorial-ball one) -- the reference breaks down on such facets
    // (SURVEY F1).  Decide membership by the exact equatorial-ball test of
    // the 3D points instead; on axis-parallel polygons both tests coincide.
    const Dev& D = *C.D;
    return equatorial_cmp_robust(PT(D, t.x), PT(D, t.y), PT(D, t.z), PT(D, C.vid)) < 0;
  }
  double pc[2];
  C.pos(t.x, pa); C.pos(t.y, pb); C.pos(t.z, pc);
  return incircle2d(pa, pb, pc, C.p) > 0;
}
__device__ __forceinline__ int t2_vert(const int4& t, int k) { return k == 0 ? t.x : (k == 1 ? t.y : t.z); }
__device__ inline int t2_nb(const Dev& D, const int4& t, int k) {   // triangle across edge k=(v_k, v_k+1)
  int a = t2_vert(t, k), b = t2_vert(t, (k + 1) % 3);
  return he_lookup(D, b, a, t.w);
}
__device__ inline int t2_add(const Dev& D, int a, int b, int c, int pid) {
  int tid = atomicAdd(&D.ctr->nt2, 1);
  if (tid >= D.t2cap) { raise_err(GQ_ERR_CAP); return -1; }
  D.t2v[tid] = make_int4(a, b, c, pid);
  D.t2alive[tid] = 1;
  if (c != GHOST) D.t2last[pid] = tid;
  ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(a, b, pid), tid);
  ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(b, c, pid), tid);
  ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(c, a, pid), tid);
  atomicAdd(D.t2count + pid, 1);
  return tid;
}

// 2D cavity of one insertion (facets.py:185-236): forced triangles + the
// Delaunay cavity of p grown from `seeds`, expanded until star-shaped, seed
// component.  Result tids in `cav` (set semantics).  Returns count or -1.
__device__ __noinline__ int tri2_cavity(const Tri2Ctx& C, const int* forced, int nforced, const int* seeds, int nseeds,
                                  ISet& set, int* cav, int* stack, int cap) {
  const Dev& D = *C.D;
  set.clear();
  int n = 0;
  atomicAdd(&D.ctr->t2st[0], 1ull);
  if (C.follow3d) {
    // Oblique polygon.  Its Steiner points round off the polygon plane, so an
    // in-plane Delaunay cavity and the 3D cavity disagree near cocircular
    // configurations; every disagreement leaves a missing subface whose split
    // makes more (a runaway the reference never meets: it stops on oblique
    // facets).  The retiling therefore follows the mesh: remove
    // exactly the subfaces the 3D cavity crossed (plus the split edge's
    // triangles) and fan p onto their rim, whose edges all lie on the 3D
    // cavity boundary -- every new subface is a face of the new star
    // (SURVEY F5's 3D-derived delta).  In-plane Delaunay quality is then
    // restored by the ordinary encroachment checks.
    nseeds = 0;
    if (nforced == 0) return 0;
  }
  // own Delaunay cavity from the first seed in region
  int seed = -1;
  for (int k = 0; k < nseeds && seed < 0; ++k)
    if (seeds[k] >= 0 && D.t2alive[seeds[k]] && D.t2v[seeds[k]].w == C.pid && tri_in_region(C, seeds[k])) seed = seeds[k];
  int start = (nseeds > 0 && seeds[0] >= 0 && D.t2alive[seeds[0]]) ? seeds[0] : -1;
  if (seed < 0 && start < 0 && nforced == 0) {
    // no hint from the 3D side (the target's triangle was retiled earlier in
    // the round): walk from the polygon's most recent triangle, like the
    // reference walks from its last touched triangle (facets.py:107-123)
    int t = D.t2last[C.pid];
    if (t >= 0 && D.t2alive[t] && D.t2v[t].w == C.pid) start = t;
  }
  if (seed < 0 && start >= 0) {
    // facets.py:107-123: walk toward p
    int tid = start;
    int n_alive = D.t2count[C.pid];
    int s = 0;
    for (; s < 4 * n_alive + 16; ++s) {
      int4 t = D.t2v[tid];
      if (t.z == GHOST) break;
      bool moved = false;
      for (int k = 0; k < 3; ++k) {
        double pu[2], pv[2];
        C.pos(t2_vert(t, k), pu); C.pos(t2_vert(t, (k + 1) % 3), pv);
        if (orient2d(pu, pv, C.p) < 0) { int nb = t2_nb(D, t, k); if (nb >= 0) { tid = nb; moved = true; } break; }
      }
      if (!moved) break;
    }
    atomicAdd(&D.ctr->t2st[1], (unsigned long long)s);
    if (tri_in_region(C, tid)) seed = tid;
    if (seed < 0 && nforced == 0) {   // exhaustive fallback (facets.py:121-123)
      const int nt2 = D.ctr->nt2;
      atomicAdd(&D.ctr->t2st[2], 1ull); atomicAdd(&D.ctr->t2st[3], (unsigned long long)nt2);
      for (int t = 0; t < nt2 && seed < 0; ++t)
        if (D.t2alive[t] && D.t2v[t].w == C.pid && tri_in_region(C, t)) seed = t;
    }
  }
  int own_seed = seed;
  if (seed >= 0) {
    cav[n] = seed; set.put(seed, n); ++n;
    int sp = 0;
    stack[sp++] = seed;
    while (sp > 0) {
      int tid = stack[--sp];
      int4 t = D.t2v[tid];
      for (int k = 0; k < 3; ++k) {
        int nb = t2_nb(D, t, k);
        if (nb < 0 || set.find(nb) >= 0) continue;
        if (tri_in_region(C, nb)) {
          if (n >= cap) return -1;
          cav[n] = nb; set.put(nb, n); ++n;
          stack[sp++] = nb;
        }
      }
    }
  } else if (nforced == 0) {
#ifdef GQ_DEBUG2D
    printf("[2d] no seed pid %d vid %d nseeds %d seed0 %d alive %d count %d p %.17g %.17g\n", C.pid, C.vid, nseeds,
           nseeds > 0 ? seeds[0] : -9, nseeds > 0 && seeds[0] >= 0 ? (int)D.t2alive[seeds[0]] : -1, D.t2count[C.pid], C.p[0], C.p[1]);
#endif
    raise_err(GQ_ERR_2D);
    return -1;
  }
  for (int k = 0; k < nforced; ++k) {
    int tid = forced[k];
    if (tid < 0 || set.find(tid) >= 0) continue;
    if (n >= cap) return -1;
    cav[n] = tid; set.put(tid, n); ++n;
  }
  if (nforced > 0) {
    // expand until star-shaped (facets.py:150-170)
    bool changed = true;
    while (changed) {
      changed = false;
      int n0 = n;
      for (int a = 0; a < n0; ++a) {
        int4 t = D.t2v[cav[a]];
        for (int k = 0; k < 3; ++k) {
          int u = t2_vert(t, k), v = t2_vert(t, (k + 1) % 3);
          if (u == GHOST || v == GHOST) continue;
          int nb = he_lookup(D, v, u, C.pid);
          if (nb < 0 || set.find(nb) >= 0) continue;
          double pu[2], pv[2];
          C.pos(u, pu); C.pos(v, pv);
          if (orient2d(pu, pv, C.p) <= 0) {
            if (n >= cap) return -1;
            cav[n] = nb; set.put(nb, n); ++n;
            changed = true;
          }
        }
      }
      if (n == D.t2count[C.pid]) {
#ifdef GQ_DEBUG2D
        printf("[2d] consumed pid %d vid %d n %d nforced %d own %d\n", C.pid, C.vid, n, nforced, own_seed);
#endif
        raise_err(GQ_ERR_2D); return -1;
      }
    }
    // component of the seed (facets.py:172-183)
    int s0 = own_seed;
    if (s0 < 0) { s0 = cav[0]; for (int a = 1; a < n; ++a) if (cav[a] < s0) s0 = cav[a]; }
    // mark component in stack[] area after cav: use set values: >=0 index; comp via second pass
    int* comp = stack + cap;   // caller provides 2*cap stack
    for (int a = 0; a < n; ++a) comp[a] = 0;
    int ks = set.find(s0);
    comp[ks] = 1;
    int sp = 0;
    stack[sp++] = s0;
    int nc = 1;
    while (sp > 0) {
      int tid = stack[--sp];
      int4 t = D.t2v[tid];
      for (int k = 0; k < 3; ++k) {
        int nb = t2_nb(D, t, k);
        if (nb < 0) continue;
        int kk = set.find(nb);
        if (kk < 0 || comp[kk]) continue;
        comp[kk] = 1; ++nc;
        stack[sp++] = nb;
      }
    }
    if (nc < n) {
      int m = 0;
      for (int a = 0; a < n; ++a) if (comp[a]) cav[m++] = cav[a];
      n = m;
      set.clear();
      for (int a = 0; a < n; ++a) set.put(cav[a], a);
    }
  }
  return n;
}

// apply a computed 2D cavity: remove its triangles, star vid onto the rim.
// Removed / added non-ghost triangle keys are reported through callbacks.
template <class FR, class FA>
__device__ inline bool tri2_apply(const Tri2Ctx& C, const int* cav, int n, ISet& set, FR on_removed, FA on_added) {
  const Dev& D = *C.D;
  // collect rim edges first (needs the old adjacency)
  int rim[3 * 256][2];
  int nr = 0;
  for (int a = 0; a < n; ++a) {
    int4 t = D.t2v[cav[a]];
    for (int k = 0; k < 3; ++k) {
      int u = t2_vert(t, k), v = t2_vert(t, (k + 1) % 3);
      int m = he_lookup(D, v, u, C.pid);
      if (m < 0 || set.find(m) < 0) {
        if (nr >= 3 * 256) { raise_err(GQ_ERR_CAP); return false; }
        rim[nr][0] = u; rim[nr][1] = v; ++nr;
      }
    }
  }
  for (int a = 0; a < n; ++a) {
    int4 t = D.t2v[cav[a]];
    D.t2alive[cav[a]] = 0;
    atomicSub(D.t2count + C.pid, 1);
    if (t.z != GHOST) on_removed(t.x, t.y, t.z);
  }
  for (int r = 0; r < nr; ++r) {
    int u = rim[r][0], v = rim[r][1];
    if (u == GHOST || v == GHOST) {
      if (u == GHOST) t2_add(D, v, C.vid, GHOST, C.pid);
      else t2_add(D, C.vid, u, GHOST, C.pid);
    } else {
      int tid = t2_add(D, u, v, C.vid, C.pid);
      on_added(u, v, C.vid, tid);
    }
  }
  return true;
}

}  // namespace gq
