// gq_main.cu -- round driver, kernels and C ABI of libgqm3d.so (sm_100a).
//
// One gq_refine() call = the reference's refine() from init_delaunay to the
// final verification scan (/root/reference/pkg/src/tetrefine/refine.py:523-925)
// with the whole mesh resident in HBM.  Each round is a fixed chain of
// data-parallel kernels over the round's candidates:
//
//   pool      phase selection + candidate construction        (refine.py:583-665)
//   regions   Delaunay region of every splitting point         (mesh.py:450-521)
//             + encroachment probe of the grown cavity -> redirects
//   filter    greedy-by-priority disjoint set as fixed-priority
//             local-minimum iterations (== growblast.greedy_oracle)
//   insert    vertex ids in priority order, facet 2D retiling in priority
//             passes, subsegment splits, Bowyer-Watson stars   (refine.py:685-737)
//   fallback  failed candidates, sequentially, on the updated mesh (refine.py:748-799)
//   post      presence + encroachment of new / dirty constraints, compaction
//
// The host reads back a handful of counters per stage; all mesh data stays
// on the device.
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "gq_dev.cuh"
#include "gq_block.cuh"
#include "gq_warp.cuh"
#include "../../include/gqm3d.h"

using namespace gq;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x); } while (0)

// candidate kinds / phases
#define K_SEG 0
#define K_FACE 1
#define K_TET 2

// candidate status
#define CS_OK 0
#define CS_CNSS 1
#define CS_TOOCLOSE 2
#define CS_MEMB 3
#define CS_OVF 4
#define CS_DROP 5      // redirected / skipped before the pool

// slab capacities (normal pass); overflowing candidates rerun with big slabs
#define CT 512
#define CF 1088
#define CC 96
#define CRD 64
#define CTB 4096
#define CFB 8200
#define CCB 2048

struct Scr {           // per-thread scratch arenas
  int* tkey; int* tval; unsigned int* tep; int tcap;
  unsigned long long* fkey; unsigned int* fep; int fcap;
  unsigned int* epoch;
  int* list; int* stack; uint8_t* in; uint8_t* comp; int cap;
  int nthreads;
};
__device__ inline Scratch scratch_for(const Scr& s, int tid) {
  Scratch S;
  S.tset.key = s.tkey + (size_t)tid * s.tcap; S.tset.val = s.tval + (size_t)tid * s.tcap;
  S.tset.ep = s.tep + (size_t)tid * s.tcap; S.tset.cur = s.epoch + 2 * tid; S.tset.cap = s.tcap;
  S.fset.key = s.fkey + (size_t)tid * s.fcap; S.fset.ep = s.fep + (size_t)tid * s.fcap;
  S.fset.cur = s.epoch + 2 * tid + 1; S.fset.cap = s.fcap;
  S.list = s.list + (size_t)tid * s.cap; S.stack = s.stack + (size_t)tid * 2 * s.cap;
  S.in = s.in + (size_t)tid * s.cap; S.comp = s.comp + (size_t)tid * s.cap; S.cap = s.cap;
  return S;
}

struct Cand {          // candidate arrays (capacity cap)
  int cap;
  int* kind; int* tgt; int* seed; int* status; int* memb; int* pool; int* rank;
  int4* allow; int* nallow; int* extra;
  double* p; unsigned long long* h; int4* canon;
  int* state; int* vid; int* nt0;
  // region slabs (normal); big slab index in bigi (-1 none)
  int* ntet; int* nbf; int* ncr; int* nbsub; int* nbseg; int* neseg; double* mind;
  int* tets; int* bf; int* cr; int* crf; int* bsub; int* bseg; int* eseg;
  int* rseg; int* rface; int* nrseg; int* nrface;
  int* bigi;
  int* btets; int* bbf; int* bcr; int* bcrf; int* bbsub; int* bbseg; int* beseg;
  int nbigcap;
};
struct SlabView { int* tets; int* bf; int* cr; int* crf; int* bsub; int* bseg; int* eseg; int ct, cf, cc; };
__device__ __forceinline__ SlabView slab(const Cand& C, int c) {
  SlabView v;
  int b = C.bigi[c];
  if (b < 0) {
    v.tets = C.tets + (size_t)c * CT; v.bf = C.bf + (size_t)c * CF; v.cr = C.cr + (size_t)c * CC;
    v.crf = C.crf + (size_t)c * CC; v.bsub = C.bsub + (size_t)c * CC; v.bseg = C.bseg + (size_t)c * CC;
    v.eseg = C.eseg + (size_t)c * CC; v.ct = CT; v.cf = CF; v.cc = CC;
  } else {
    v.tets = C.btets + (size_t)b * CTB; v.bf = C.bbf + (size_t)b * CFB; v.cr = C.bcr + (size_t)b * CCB;
    v.crf = C.bcrf + (size_t)b * CCB; v.bsub = C.bbsub + (size_t)b * CCB; v.bseg = C.bbseg + (size_t)b * CCB;
    v.eseg = C.beseg + (size_t)b * CCB; v.ct = CTB; v.cf = CFB; v.cc = CCB;
  }
  return v;
}

__device__ unsigned long long g_region_calls;
__device__ unsigned long long g_tested;       // tets tested for membership (algorithmic bytes)

// ---------------------------------------------------------------------------
// priorities (refine.py:35-52)
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x = x + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ inline unsigned long long prio_hash(const int* canon, int n, int round_no, unsigned long long seed) {
  unsigned long long h = splitmix64(seed ^ ((unsigned long long)round_no * 0x9E3779B97F4A7C15ull));
  for (int k = 0; k < n; ++k) h = splitmix64(h ^ (unsigned long long)((long long)canon[k] + 2));
  return h;
}

// ---------------------------------------------------------------------------
// skipped-element log
struct SkipLog { int* rows; int cap; };   // 8 ints: round, kind, reason, n, v0..v3
__device__ __noinline__ void log_skip(const Dev& D, const SkipLog& L, int round_no, int kind, int reason, const int* v, int n) {
  int k = atomicAdd(&D.ctr->nskip, 1);
  if (k >= L.cap) { raise_err(GQ_ERR_CAP); return; }
  int* r = L.rows + 8 * (size_t)k;
  r[0] = round_no; r[1] = kind; r[2] = reason; r[3] = n;
  for (int i = 0; i < 4; ++i) r[4 + i] = i < n ? v[i] : -1;
}
__device__ inline void tet_canon(const Dev& D, int t, int* c) {
  int4 q = D.tv[t];
  c[0] = q.x; c[1] = q.y; c[2] = q.z; c[3] = q.w;
  for (int a = 1; a < 4; ++a) { int x = c[a], b = a - 1; while (b >= 0 && c[b] > x) { c[b + 1] = c[b]; --b; } c[b + 1] = x; }
}

// ---------------------------------------------------------------------------
// candidate construction (refine.py:338-375)
struct CandCtx { int round_no; unsigned long long seed; int with_facets; };

__device__ __noinline__ int walk_seed(const Dev& D, const double* p, int near_vertex) {   // refine.py:416-418
  int hint = D.vert_tet[near_vertex];
  return walk(D, p, hint >= 0 ? hint : -1);
}

// fills point / priority / seed / allowed pids / claim extra for candidate c.
// Returns false when the element is degenerate (DegenerateTet / DegenerateTri).
__device__ __noinline__ bool make_cand(const Dev& D, const Cand& C, int c, const CandCtx& X, Scratch& S) {
  int kind = C.kind[c], tgt = C.tgt[c];
  double* p = C.p + 3 * (size_t)c;
  int canon[4];
  int nc = 0;
  C.seed[c] = -1; C.nallow[c] = 0; C.extra[c] = -1;
  if (kind == K_TET) {
    tet_canon(D, tgt, canon); nc = 4;
    int4 q = D.tv[tgt];
    Sphere s;
    if (circumsphere_tet(PT(D, q.x), PT(D, q.y), PT(D, q.z), PT(D, q.w), s) != 0) return false;
    p[0] = s.c[0]; p[1] = s.c[1]; p[2] = s.c[2];
  } else if (kind == K_SEG) {
    int2 e = D.sg_uv[tgt];
    canon[0] = e.x; canon[1] = e.y; nc = 2;
    const double *pu = PT(D, e.x), *pv = PT(D, e.y);
    for (int k = 0; k < 3; ++k) p[k] = (pu[k] + pv[k]) / 2.0;
    if (!edge_exists(D, e.x, e.y, S.tset, S.stack, 2 * S.cap)) C.seed[c] = walk_seed(D, p, e.x);
    if (X.with_facets) {
      int sid = D.sg_sid[tgt];
      int o0 = D.segpoly_off[sid], o1 = D.segpoly_off[sid + 1];
      int na = 0;
      int4 al = make_int4(-1, -1, -1, -1);
      for (int o = o0; o < o1 && na < 4; ++o) {
        int pid = D.segpoly[o];
        if (na == 0) al.x = pid; else if (na == 1) al.y = pid; else if (na == 2) al.z = pid; else al.w = pid;
        ++na;
      }
      if (o1 - o0 > 4) raise_err(GQ_ERR_CAP);
      C.allow[c] = al; C.nallow[c] = na;
      C.extra[c] = tgt;
    }
  } else {
    int4 f = D.sf_v[tgt];
    canon[0] = f.x; canon[1] = f.y; canon[2] = f.z; nc = 3;
    Sphere s;
    if (!circumcircle_tri(PT(D, f.x), PT(D, f.y), PT(D, f.z), s)) return false;
    p[0] = s.c[0]; p[1] = s.c[1]; p[2] = s.c[2];
    int slot = find_face(D, f.x, f.y, f.z, S.tset, S.stack, 2 * S.cap);
    if (slot < 0) C.seed[c] = walk_seed(D, p, f.x);
    C.allow[c] = make_int4(f.w, -1, -1, -1); C.nallow[c] = 1;
    if (slot >= 0) C.extra[c] = min(slot, tnk(D, slot >> 2, slot & 3));
  }
  C.h[c] = prio_hash(canon, nc, X.round_no, X.seed);
  int4 cn = make_int4(nc > 0 ? canon[0] : INT_MAX, nc > 1 ? canon[1] : INT_MAX, nc > 2 ? canon[2] : INT_MAX,
                      nc > 3 ? canon[3] : INT_MAX);
  C.canon[c] = cn;
  return true;
}

__device__ inline Allow allow_of(const Cand& C, int c) {
  Allow A;
  A.n = C.nallow[c];
  int4 a = C.allow[c];
  A.pid[0] = a.x; A.pid[1] = a.y; A.pid[2] = a.z; A.pid[3] = a.w;
  return A;
}

// seeds of a candidate (mesh.py:416-433): tet itself / sorted edge ring /
// the two tets of the subface, or the walk seed of a missing constraint
__device__ __noinline__ int cand_seeds(const Dev& D, const Cand& C, int c, int* out, Scratch& S) {
  if (C.seed[c] >= 0) { out[0] = C.seed[c]; return 1; }
  int kind = C.kind[c], tgt = C.tgt[c];
  DCHK(kind >= 0 && kind <= 2);
  if (kind == K_TET) { out[0] = tgt; return 1; }
  if (kind == K_SEG) {
    int2 e = D.sg_uv[tgt];
    int n = 0;
    around_vertex(D, e.x, S.tset, S.stack, 2 * S.cap, [&](int t) {
      if (has_v(D.tv[t], e.y)) {
        if (n < 32) out[n++] = t;
        else { int mx = 0; for (int k = 1; k < 32; ++k) if (out[k] > out[mx]) mx = k; if (t < out[mx]) out[mx] = t; }
      }
      return false;
    });
    for (int a = 1; a < n; ++a) { int x = out[a], b = a - 1; while (b >= 0 && out[b] > x) { out[b + 1] = out[b]; --b; } out[b + 1] = x; }
    return n;
  }
  int4 f = D.sf_v[tgt];
  int slot = find_face(D, f.x, f.y, f.z, S.tset, S.stack, 2 * S.cap);
  if (slot < 0) return 0;
  int t = slot >> 2, u = tnk(D, t, slot & 3) >> 2;
  if (u >= 0 && D.alive[u]) { out[0] = min(t, u); out[1] = max(t, u); return 2; }
  out[0] = t;
  return 1;
}

__device__ inline RegionOut region_view(const Cand& C, int c, const SlabView& v, int probe) {
  RegionOut O;
  O.tets = v.tets; O.bf = v.bf; O.cr = v.cr; O.crf = v.crf; O.bsub = v.bsub; O.bseg = v.bseg; O.eseg = v.eseg;
  O.ctet = v.ct; O.cbf = v.cf; O.ccon = v.cc;
  O.probe = probe;
  O.rseg = C.rseg + (size_t)c * CRD; O.rface = C.rface + (size_t)c * CRD; O.crd = CRD;
  O.nrseg = 0; O.nrface = 0;
  O.memb = -1; O.seed = -1;
  return O;
}
__device__ inline void store_region(const Cand& C, int c, const RegionOut& O) {
  C.ntet[c] = O.ntet; C.nbf[c] = O.nbf; C.ncr[c] = O.ncr; C.nbsub[c] = O.nbsub; C.nbseg[c] = O.nbseg;
  C.neseg[c] = O.neseg; C.mind[c] = O.mind; C.nrseg[c] = O.nrseg; C.nrface[c] = O.nrface;
}

// ===========================================================================
// kernels
// ===========================================================================

__global__ void k_make_cands(Dev D, Cand C, Scr SC, int n0, int n1, CandCtx X, SkipLog L, double lmin2) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  for (int c = n0 + tid; c < n1; c += gridDim.x * blockDim.x) {
    C.status[c] = CS_OK;
    C.bigi[c] = -1;
    bool ok = make_cand(D, C, c, X, S);
    if (C.kind[c] == K_TET) {
      int t = C.tgt[c];
      if (!ok) {
        D.skip[t] = 1;
        int cv[4]; tet_canon(D, t, cv);
        log_skip(D, L, X.round_no, K_TET, 0, cv, 4);
        C.status[c] = CS_DROP;
        continue;
      }
      int4 q = D.tv[t];
      Sphere s;
      circumsphere_tet(PT(D, q.x), PT(D, q.y), PT(D, q.z), PT(D, q.w), s);
      if (s.r2 < lmin2) {
        D.skip[t] = 1;
        int cv[4]; tet_canon(D, t, cv);
        log_skip(D, L, X.round_no, K_TET, 1, cv, 4);
        C.status[c] = CS_DROP;
      }
    } else if (!ok) {
      raise_err(GQ_ERR_DEGEN);
      C.status[c] = CS_DROP;
    }
  }
}

// region of every candidate in [n0,n1) with status OK (or the listed ones)
__global__ void k_region(Dev D, Cand C, Scr SC, int n0, int n1, const int* list, int probe, int big) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  int n = list ? n1 : n1 - n0;
  for (int w = tid; w < n; w += gridDim.x * blockDim.x) {
    int c = list ? list[w] : n0 + w;   // with a list, n0 is the first big slab
    if (C.status[c] != CS_OK && !(big && C.status[c] == CS_OVF)) continue;
    if (big) C.bigi[c] = n0 + w;
    SlabView v = slab(C, c);
    int seeds[32];
    int ns = cand_seeds(D, C, c, seeds, S);
    int pr = probe;
    if (pr == 3) pr = C.kind[c] == K_TET ? 2 : (C.kind[c] == K_FACE ? 1 : 0);
    RegionOut O = region_view(C, c, v, pr);
    atomicAdd(&g_region_calls, 1ull);
    int st = ns == 0 ? RS_CNSS : region_compute(D, C.p + 3 * (size_t)c, seeds, ns, allow_of(C, c), S, O);
    store_region(C, c, O);
    if (st == RS_OK) atomicAdd(&g_tested, (unsigned long long)(O.ntet + O.nbf));
    if (st == RS_OK) {
      C.status[c] = (O.mind <= D.too_close_sq) ? CS_TOOCLOSE : CS_OK;
    } else if (st == RS_OVERFLOW) {
      C.status[c] = big ? CS_CNSS : CS_OVF;
      if (big) raise_err(GQ_ERR_CAP);
    } else if (st == RS_MEMBRANE) {
      C.status[c] = CS_MEMB; C.memb[c] = O.memb;
    } else {
      C.status[c] = CS_CNSS;
    }
  }
}

// coarse grid of inserted vertices: a pending point's first walk starts next
// to an already inserted vertex instead of at the initial tet
struct CellHint { double lo[3], inv[3]; int G; int* cellv; };
__device__ __forceinline__ int cell_of(const CellHint& H, const double* p) {
  int c[3];
  for (int k = 0; k < 3; ++k) {
    double f = (p[k] - H.lo[k]) * H.inv[k];
    c[k] = f >= 0.0 ? (f < (double)H.G ? (int)f : H.G - 1) : 0;
  }
  return (c[0] * H.G + c[1]) * H.G + c[2];
}
__global__ void k_init_cellmark(Dev D, CellHint H, const int* pend, const int* plist, const int* acc, int nw) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    if (acc[w]) { int v = pend[plist[w]]; H.cellv[cell_of(H, PT(D, v))] = v; }
}
// one warp per candidate (the common case); overflowing cavities are marked
// CS_OVF for the block kernel
#define INIT_BLOCK_ROUTE 192   // bulk construction: cached cavities above this go to the block kernel
// tiers of the warp region kernel.  Measured on C2: a 128-tet tier at 16 warps
// / SM plus the 512-tet tier for its overflows is no faster than the 512-tet
// tier alone (the 4% large cavities cost what the occupancy gains), so both
// tiers are the large one and the second pass is skipped.
#define WT1_MAXT 512
#define WT1_HASH 2048
#define WT1_MINB 1
#define WT2_MAXT 512
#define WT2_HASH 2048
typedef WarpSharedT<WT1_MAXT, WT1_HASH> WarpShared1;
typedef WarpSharedT<WT2_MAXT, WT2_HASH> WarpShared2;
// candidates [n0,n1) (list == nullptr) or list[n0..n1) (the small tier's overflows)
template <int MAXT, int HASH, int MINB>
__global__ void __launch_bounds__(32 * WR_WARPS, MINB) k_region_warp(Dev D, Cand C, Scr SC, int n0, int n1, const int* list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typedef WarpSharedT<MAXT, HASH> WS;
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WS& W = reinterpret_cast<WS*>(smem_raw)[wib];
  const int gw = blockIdx.x * WR_WARPS + wib, nw = gridDim.x * WR_WARPS;
  Scratch S = scratch_for(SC, gw);
  for (int k = n0 + gw; k < n1; k += nw) {
    const int c = list ? list[k] : k;
    if (C.status[c] != (list ? CS_OVF : CS_OK)) continue;
    DCHK(C.bigi[c] == -1);
    if (lane == 0) W.nseeds = cand_seeds(D, C, c, W.seeds, S);
    __syncwarp();
    int ns = W.nseeds;
    DCHK(ns >= 0 && ns <= 32);
    SlabView v = slab(C, c);
    RegionOut O = region_view(C, c, v, 0);
    int st = ns == 0 ? RS_CNSS : region_warp(D, C.p + 3 * (size_t)c, W.seeds, ns, allow_of(C, c), W, S, O);
    if (lane == 0) {
      atomicAdd(&g_region_calls, 1ull);
      store_region(C, c, O);
      if (st == RS_OK) {
        atomicAdd(&g_tested, (unsigned long long)(O.ntet + O.nbf));
        C.status[c] = (O.mind <= D.too_close_sq) ? CS_TOOCLOSE : CS_OK;
      } else if (st == RS_OVERFLOW) C.status[c] = CS_OVF;
      else if (st == RS_MEMBRANE) { C.status[c] = CS_MEMB; C.memb[c] = O.memb; }
      else C.status[c] = CS_CNSS;
    }
    __syncwarp();
  }
}
// bulk construction, warp per pending point (cached cavities re-validated);
// redo_ovf: the large tier, run on the small tier's overflows
template <int MAXT, int HASH, int MINB>
__global__ void __launch_bounds__(32 * WR_WARPS, MINB) k_init_region_warp(Dev D, Cand C, Scr SC, const int* pend, const int* plist,
                                                                    int Wn, int* hint, const int* succ, const int* touched, int round,
                                                                    CellHint H, int redo_ovf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typedef WarpSharedT<MAXT, HASH> WS;
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WS& W = reinterpret_cast<WS*>(smem_raw)[wib];
  const int gw = blockIdx.x * WR_WARPS + wib, nw = gridDim.x * WR_WARPS;
  Scratch S = scratch_for(SC, gw);
  for (int w = gw; w < Wn; w += nw) {
    int c = plist[w];
    if (lane == 0 && g_wdbg) { g_wdbg[2 * gw] = c; g_wdbg[2 * gw + 1] = 0; }
    DCHK(c >= 0 && c < C.cap);
    int st0 = C.status[c];
    if ((st0 == CS_OVF) != (redo_ovf != 0)) continue;
    if (st0 == CS_OK && C.memb[c] >= 0) {
      SlabView v = slab(C, c);
      bool bad = false;
      for (int k = lane; k < C.ntet[c]; k += 32) {
        int t = v.tets[k];
        if (!D.alive[t] || touched[t] >= C.memb[c]) bad = true;
      }
      if (!__any_sync(0xffffffffu, bad)) continue;
    }
    // a point whose last cavity was large (a box corner far outside the current
    // hull, recomputed every round while it waits) goes straight to the block
    // kernel, which grows it with 256 threads instead of 32
    if (!redo_ovf && st0 == CS_OK && (C.memb[c] == -2 || (C.memb[c] >= 0 && C.ntet[c] > INIT_BLOCK_ROUTE))) {
      if (lane == 0) { C.status[c] = CS_OVF; C.memb[c] = -1; }
      __syncwarp();
      continue;
    }
    int vtx = pend[c];
    if (lane == 0 && g_wdbg) { g_wdbg[2 * gw] = c; g_wdbg[2 * gw + 1] = 1; }
    DCHK(vtx >= 0 && vtx < D.vcap);
    const double* p = PT(D, vtx);
    if (lane == 0) {
      int h = hint[c];
      DCHK(h >= -1 && h < D.tcap);
      if (h < 0) {                      // first walk: start beside a nearby inserted vertex
        int cv = H.cellv[cell_of(H, p)];
        h = cv >= 0 ? D.vert_tet[cv] : 0;
      }
      while (h >= 0 && !D.alive[h]) h = succ[h];
      // a ghost hint (last seen outside the hull) restarts at the hull tet behind
      // it: walk() would otherwise rescan the tet array for a real tet.  The
      // unconstrained cavity does not depend on the seed.
      if (h >= 0 && D.tv[h].w == GHOST) h = tnk(D, h, 3) >> 2;
      int t = walk(D, p, h);
      hint[c] = t;
      W.seeds[0] = t;
    }
    __syncwarp();
    SlabView sv = slab(C, c);
    RegionOut O = region_view(C, c, sv, 0);
    Allow A; A.n = 0;
    if (lane == 0 && g_wdbg) g_wdbg[2 * gw + 1] = 2;
    int r = region_warp(D, p, W.seeds, 1, A, W, S, O, true);
    if (lane == 0 && g_wdbg) g_wdbg[2 * gw + 1] = 99;
    if (lane == 0) {
      atomicAdd(&g_region_calls, 1ull);
      store_region(C, c, O);
      C.extra[c] = -1; C.kind[c] = K_TET; C.rank[c] = c; C.memb[c] = round;
      if (r == RS_OK) { C.status[c] = CS_OK; atomicAdd(&g_tested, (unsigned long long)(O.ntet + O.nbf)); }
      else if (r == RS_OVERFLOW) { C.status[c] = CS_OVF; C.memb[c] = -1; }
      else { C.status[c] = CS_CNSS; raise_err(GQ_ERR_DEGEN); }
    }
    __syncwarp();
  }
}

// oversized cavities: one block per candidate (threads in proportion to
// region size); big slabs base+w
__global__ void __launch_bounds__(BR_THREADS) k_region_block(Dev D, Cand C, Scr SB, const int* list, int nb, int base) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BlockShared& B = *reinterpret_cast<BlockShared*>(smem_raw);
  Scratch S = scratch_for(SB, blockIdx.x);
  for (int w = blockIdx.x; w < nb; w += gridDim.x) {
    int c = list[w];
    if (threadIdx.x == 0) C.bigi[c] = base + w;
    __syncthreads();
    SlabView v = slab(C, c);
    __shared__ int s_seeds[32];
    __shared__ int s_ns;
    if (threadIdx.x == 0) s_ns = cand_seeds(D, C, c, s_seeds, S);
    __syncthreads();
    RegionOut O = region_view(C, c, v, 0);
    int st = s_ns == 0 ? RS_CNSS : region_block(D, C.p + 3 * (size_t)c, s_seeds, s_ns, allow_of(C, c), B, S, O);
    if (threadIdx.x == 0) {
      atomicAdd(&g_region_calls, 1ull);
      store_region(C, c, O);
      if (st == RS_OK) {
        atomicAdd(&g_tested, (unsigned long long)(O.ntet + O.nbf));
        C.status[c] = (O.mind <= D.too_close_sq) ? CS_TOOCLOSE : CS_OK;
      } else if (st == RS_OVERFLOW) { C.status[c] = CS_CNSS; raise_err(GQ_ERR_CAP); }
      else if (st == RS_MEMBRANE) { C.status[c] = CS_MEMB; C.memb[c] = O.memb; }
      else C.status[c] = CS_CNSS;
    }
    __syncthreads();
  }
}
__global__ void __launch_bounds__(BR_THREADS) k_init_region_block(Dev D, Cand C, Scr SB, const int* pend, const int* list, int nb,
                                                                  int* hint, const int* succ, int round) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BlockShared& B = *reinterpret_cast<BlockShared*>(smem_raw);
  Scratch S = scratch_for(SB, blockIdx.x);
  for (int w = blockIdx.x; w < nb; w += gridDim.x) {
    int c = list[w];
    __shared__ int s_t;
    if (threadIdx.x == 0) {
      C.bigi[c] = w;
      const double* p = PT(D, pend[c]);
      int h = hint[c];
      if (h < 0) h = 0;
      while (h >= 0 && !D.alive[h]) h = succ[h];
      if (h >= 0 && D.tv[h].w == GHOST) h = tnk(D, h, 3) >> 2;
      s_t = walk(D, p, h);
      hint[c] = s_t;
    }
    __syncthreads();
    SlabView v = slab(C, c);
    RegionOut O = region_view(C, c, v, 0);
    int seeds[1] = {s_t};
    Allow A; A.n = 0;
    int st = region_block(D, PT(D, pend[c]), seeds, 1, A, B, S, O);
    if (threadIdx.x == 0) {
      atomicAdd(&g_region_calls, 1ull);
      store_region(C, c, O);
      C.extra[c] = -1; C.kind[c] = K_TET; C.rank[c] = c; C.memb[c] = round;
      if (st == RS_OK) { C.status[c] = CS_OK; atomicAdd(&g_tested, (unsigned long long)(O.ntet + O.nbf)); }
      else if (st == RS_OVERFLOW) { C.status[c] = CS_OVF; C.memb[c] = -1; raise_err(GQ_ERR_CAP); }
      else { C.status[c] = CS_CNSS; raise_err(GQ_ERR_DEGEN); }
    }
    __syncthreads();
  }
}

// redirect decision (refine.py:595-613, 615-662); marks records RF_REDIR
__global__ void k_redirect(Dev D, Cand C, int n0, int n1, int* nredir) {
  for (int c = n0 + blockIdx.x * blockDim.x + threadIdx.x; c < n1; c += gridDim.x * blockDim.x) {
    int kind = C.kind[c];
    if (kind == K_SEG || C.status[c] == CS_DROP) continue;
    int ns = C.nrseg[c], nf = C.nrface[c];
    if (ns > 0) {
      for (int k = 0; k < ns; ++k) atomicOr(D.sg_fl + C.rseg[(size_t)c * CRD + k], RF_REDIR);
      atomicAdd(nredir, 1);
      C.status[c] = CS_DROP;
    } else if (kind == K_TET && nf > 0) {
      for (int k = 0; k < nf; ++k) atomicOr(D.sf_fl + C.rface[(size_t)c * CRD + k], RF_REDIR);
      atomicAdd(nredir + 1, 1);
      C.status[c] = CS_DROP;
    } else if (kind == K_TET) {
      // refine.py:378-413 hull-exit walk from the tet toward its circumcentre
      int t = C.tgt[c];
      const double* p = C.p + 3 * (size_t)c;
      int cur = t, prev = -1;
      int max_steps = walk_cap(D, 64);
      int hull = -2;   // -2 none, >=0 face rec, -1 not a subface
      bool done = false;
      for (int step = 0; step < max_steps && !done; ++step) {
        int4 q = D.tv[cur];
        if (q.w == GHOST) {
          int a = q.x, b = q.y, cc = q.z; sort3(a, b, cc);
          hull = face_lookup(D, a, b, cc); done = true; break;
        }
        bool moved = false;
        for (int k = 0; k < 4; ++k) {
          int i = (k + step) & 3;
          int u = tnk(D, cur, i) >> 2;
          if (u == prev) continue;
          int f[3]; face_verts(q, i, f);
          if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) > 0) {
            if (D.tv[u].w == GHOST) {
              sort3(f[0], f[1], f[2]);
              hull = face_lookup(D, f[0], f[1], f[2]); done = true; break;
            }
            prev = cur; cur = u; moved = true; break;
          }
        }
        if (done) break;
        if (!moved) { hull = -2; done = true; break; }
      }
      if (!done) {
        int end = walk(D, p, t);
        if (end >= 0 && D.tv[end].w == GHOST) {
          int4 q = D.tv[end];
          int a = q.x, b = q.y, cc = q.z; sort3(a, b, cc);
          hull = face_lookup(D, a, b, cc);
        }
      }
      if (hull >= 0 && !(D.sf_fl[hull] & RF_SKIP)) {
        atomicOr(D.sf_fl + hull, RF_REDIR);
        atomicAdd(nredir + 1, 1);
        C.status[c] = CS_DROP;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// constraint-ball grid: the reference's ConstraintIndex (refine.py:107-253)
// on the device.  Every live subsegment / subface ball is linked into the
// uniform cells its bounding box overlaps (balls spanning > 64 cells go to a
// side list).  Queries enumerate candidates; decisions are the exact open-ball
// predicates.  Records are only appended, so registration is incremental and
// dead records are skipped at query time.
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
__global__ void k_grid_build(Dev D, CGrid g, int nseg, int nface, int pass) {
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
// post_round part 1 (refine.py:818-828): new vertices against all balls
__global__ void k_grid_newverts(Dev D, CGrid g, int v0, int v1) {
  for (int v = v0 + blockIdx.x * blockDim.x + threadIdx.x; v < v1; v += gridDim.x * blockDim.x) {
    grid_encroached(D, g, PT(D, v), 3, [&](int kind, int r) {
      unsigned int* fl = kind == 0 ? D.sg_fl + r : D.sf_fl + r;
      if (!(*fl & RF_SKIP)) atomicOr(fl, RF_ENC);
    });
  }
}
// redirect hits of candidate points (refine.py:603-613, 636-654)
__global__ void k_grid_cands(Dev D, CGrid g, Cand C, int n0, int n1) {
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

// ---------------------------------------------------------------------------
// filter: fixed-priority local-minimum iterations == greedy_oracle
struct Owners { int* own; int toff, foff, soff; };   // [tets | faces (4*tcap) | seg records]

template <class F>
__device__ inline void for_claims(const Dev& D, const Cand& C, const Owners& W, int c, F f) {
  SlabView v = slab(C, c);
  int nt = C.ntet[c], nb = C.nbf[c], ncr = C.ncr[c], nbs = C.nbseg[c], nes = C.neseg[c];
  for (int k = 0; k < nt; ++k) f(W.toff + v.tets[k]);
  for (int k = 0; k < nb; ++k) {
    int t = v.bf[k] >> 2, i = v.bf[k] & 3;
    f(W.foff + min(v.bf[k], tnk(D, t, i)));
  }
  for (int k = 0; k < ncr; ++k) f(W.foff + v.crf[k]);
  for (int k = 0; k < nbs; ++k) if (v.bseg[k] >= 0) f(W.soff + v.bseg[k]);
  for (int k = 0; k < nes; ++k) if (v.eseg[k] >= 0) f(W.soff + v.eseg[k]);
  int ex = C.extra[c];
  if (ex >= 0) f((C.kind[c] == K_SEG ? W.soff : W.foff) + ex);
}

__global__ void k_claim(Dev D, Cand C, Owners W, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 0) continue;
    int r = C.rank[c];
    for_claims(D, C, W, c, [&](int k) { atomicMin(W.own + k, r); });
  }
}
__global__ void k_decide(Dev D, Cand C, Owners W, int n, int it) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 0) continue;
    int r = C.rank[c];
    bool win = true;
    for_claims(D, C, W, c, [&](int k) { if (W.own[k] != r) win = false; });
    if (win) C.state[c] = 10 + it;   // accepted this iteration (marked next)
  }
}
__global__ void k_mark(Dev D, Cand C, Owners W, int n, int it) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 10 + it) continue;
    for_claims(D, C, W, c, [&](int k) { W.own[k] = -1; });
    C.state[c] = 1;
  }
}
__global__ void k_reject(Dev D, Cand C, Owners W, int n, int* undecided) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 0) continue;
    bool hit = false;
    for_claims(D, C, W, c, [&](int k) { if (W.own[k] == -1) hit = true; });
    if (hit) C.state[c] = 2;
    else atomicAdd(undecided, 1);
  }
}
// The same iterations as one persistent cooperative kernel: a warp per
// candidate walks its claim keys lane-parallel (contiguous slab reads), the five
// passes of an iteration are separated by grid-wide barriers, and the loop ends
// on the device when nothing is undecided -- no launches or host syncs per
// iteration.  States: 0 undecided, 1 accepted, 2 rejected, 4 rejected in the
// current iteration (claims still to release), 10+it accepted in iteration it.
template <class F>
__device__ __forceinline__ void warp_claims(const Dev& D, const Cand& C, const Owners& W, int c, int lane, F f) {
  SlabView v = slab(C, c);
  const int nt = C.ntet[c], nb = C.nbf[c], ncr = C.ncr[c], nbs = C.nbseg[c], nes = C.neseg[c];
  const int ex = C.extra[c];
  const int e1 = nt, e2 = e1 + nb, e3 = e2 + ncr, e4 = e3 + nbs, e5 = e4 + nes, tot = e5 + (ex >= 0);
  for (int j = lane; j < tot; j += 32) {
    int key;
    if (j < e1) key = W.toff + v.tets[j];
    else if (j < e2) { int b = v.bf[j - e1]; key = W.foff + min(b, tnk(D, b >> 2, b & 3)); }
    else if (j < e3) key = W.foff + v.crf[j - e2];
    else if (j < e4) { int r = v.bseg[j - e3]; if (r < 0) continue; key = W.soff + r; }
    else if (j < e5) { int r = v.eseg[j - e4]; if (r < 0) continue; key = W.soff + r; }
    else key = (C.kind[c] == K_SEG ? W.soff : W.foff) + ex;
    f(key);
  }
}
__global__ void __launch_bounds__(256) k_filter_coop(Dev D, Cand C, Owners W, int n, int* ctr) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const unsigned FULL = 0xffffffffu;
  for (int it = 0;; ++it) {
    if (gw == 0 && lane == 0) ctr[(it + 1) % 3] = 0;
    for (int c = gw; c < n; c += nw) {                       // claim
      if (C.state[c] != 0) continue;
      const int r = C.rank[c];
      warp_claims(D, C, W, c, lane, [&](int k) { atomicMin(W.own + k, r); });
    }
    grid.sync();
    for (int c = gw; c < n; c += nw) {                       // decide
      if (C.state[c] != 0) continue;
      const int r = C.rank[c];
      bool win = true;
      warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] != r) win = false; });
      win = __all_sync(FULL, win);
      if (win && lane == 0) C.state[c] = 10 + it;
    }
    grid.sync();
    for (int c = gw; c < n; c += nw) {                       // mark
      if (C.state[c] != 10 + it) continue;
      warp_claims(D, C, W, c, lane, [&](int k) { W.own[k] = -1; });
      __syncwarp();
      if (lane == 0) C.state[c] = 1;
    }
    grid.sync();
    int und = 0;
    for (int c = gw; c < n; c += nw) {                       // reject
      if (C.state[c] != 0) continue;
      bool hit = false;
      warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] == -1) hit = true; });
      hit = __any_sync(FULL, hit);
      if (lane == 0) { if (hit) C.state[c] = 4; else ++und; }
    }
    if (lane == 0 && und) atomicAdd(ctr + it % 3, und);
    grid.sync();
    for (int c = gw; c < n; c += nw) {                       // release the claims of losers
      const int st = C.state[c];
      if (st != 0 && st != 4) continue;
      warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] >= 0) W.own[k] = INT_MAX; });
      __syncwarp();
      if (st == 4 && lane == 0) C.state[c] = 2;
    }
    grid.sync();
    if (*(volatile int*)(ctr + it % 3) == 0) break;
    if (it >= 100000) {                 // safety net: the iteration always makes progress
      if (gw == 0 && lane == 0) raise_err(GQ_ERR_CAP);
      break;
    }
  }
  for (int c = gw; c < n; c += nw) {                         // clear all owner slots touched
    const int st = C.state[c];
    if (st < 0 || st == 3) continue;
    warp_claims(D, C, W, c, lane, [&](int k) { W.own[k] = INT_MAX; });
  }
}
__global__ void k_strict_state(Cand C, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (C.state[c] == 10) C.state[c] = 1;
    else if (C.state[c] == 0) C.state[c] = 2;
}
__global__ void k_reset_claims(Dev D, Cand C, Owners W, int n, int all) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    int s = C.state[c];
    if (!all && s != 0 && s != 2) continue;
    if (all && (s < 0 || s == 3)) continue;
    for_claims(D, C, W, c, [&](int k) { if (all || W.own[k] >= 0) W.own[k] = INT_MAX; });
  }
}

// ---------------------------------------------------------------------------
// insertion of the accepted set
struct Ins {          // inserted candidates in priority order
  int* list; int n;
  int nv0, nt0base;
};

// vertex ids / points / subsegment splits (refine.py:688-708 bookkeeping)
__global__ void k_ins_vertices(Dev D, Cand C, Ins I) {
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

__global__ void k_ins_segsplit(Dev D, Cand C, Ins I) {
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
    if (t >= 0 && nf < cap) forced[nf++] = t;
  }
  if (C.kind[c] == K_SEG) {   // split edge triangles (facets.py:310-315)
    int2 e = D.sg_uv[C.tgt[c]];
    int t1 = he_lookup(D, e.x, e.y, pid); if (t1 >= 0 && nf < cap) forced[nf++] = t1;
    int t2 = he_lookup(D, e.y, e.x, pid); if (t2 >= 0 && nf < cap) forced[nf++] = t2;
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
__device__ void t2_compute_body(const Dev& D, const Cand& C, const T2Items& T, Scratch& S, int start, int stride) {
  for (int w = start; w < T.n; w += stride) {
    if (T.state[w] != 0) continue;
    int c = T.cand[w], pid = T.pid[w];
    Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = C.vid[c];
    proj2(D, pid, C.p + 3 * (size_t)c, X.p);
    int forced[CC + 2]; int nf;
    t2_forced(D, C, c, pid, forced, nf, CC + 2);
    int seeds[CC + 3]; int ns = 0;
    for (int k = 0; k < nf; ++k) seeds[ns++] = forced[k];
    int ts = t2_seed_of(D, C, c, pid);
    if (ts >= 0) seeds[ns++] = ts;
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
__device__ void t2_claim_body(const Dev& D, const Cand& C, const T2Items& T, int start, int stride) {
  for (int w = start; w < T.n; w += stride) {
    if (T.state[w] != 0) continue;
    int r = C.rank[T.cand[w]];
    t2_for_claims(D, T, w, [&](int tid) { atomicMin(T.own + tid, r); });
  }
}
__device__ void t2_apply_body(const Dev& D, const Cand& C, const T2Items& T, int* applied, int start, int stride) {
  for (int w = start; w < T.n; w += stride) {
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
__device__ void t2_commit_body(const Dev& D, const Cand& C, const T2Items& T, Scratch& S, int start, int stride) {
  for (int w = start; w < T.n; w += stride) {
    if (T.state[w] != 2) continue;
    int c = T.cand[w], pid = T.pid[w];
    Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = C.vid[c];
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
      [&](int a, int b, int cc, int t2) {  // added, unless a collinear sliver
        if (collinear_sliver(D, a, b, cc)) return;
        int a0 = a, b0 = b, c0 = cc; sort3(a0, b0, c0);
        if (face_lookup(D, a0, b0, c0) >= 0) return;   // never add a key twice
        new_face_record(D, a0, b0, c0, pid, RF_LIVE | RF_CHECK);
      });
    T.nrem[w] = nrem;
    T.state[w] = 1;
  }
}
__device__ void t2_reset_body(const Dev& D, const T2Items& T, int final_pass, int start, int stride) {
  for (int w = start; w < T.n; w += stride) {
    if (!final_pass && T.state[w] == 1 && T.ncav[w] < 0) continue;
    t2_for_claims(D, T, w, [&](int tid) { T.own[tid] = INT_MAX; });
  }
}
// retire the removed subface records (after every pass, so lookups in later
// passes still see the pre-round tables only for untouched keys)
__device__ void t2_retire_body(const Dev& D, const T2Items& T, int start, int stride) {
  for (int w = start; w < T.n; w += stride) {
    const int* rem = T.rem + (size_t)w * T.rcap;
    for (int k = 0; k < T.nrem[w]; ++k) D.sf_fl[rem[k]] = 0;
  }
}

#define GRID_START (blockIdx.x * blockDim.x + threadIdx.x)
#define GRID_STRIDE (gridDim.x * blockDim.x)
__global__ void k_t2_compute(Dev D, Cand C, T2Items T, Scr SC) {
  Scratch S = scratch_for(SC, GRID_START);
  t2_compute_body(D, C, T, S, GRID_START, GRID_STRIDE);
}
__global__ void k_t2_claim(Dev D, Cand C, T2Items T) { t2_claim_body(D, C, T, GRID_START, GRID_STRIDE); }
__global__ void k_t2_apply(Dev D, Cand C, T2Items T, Scr SC, int* applied) { t2_apply_body(D, C, T, applied, GRID_START, GRID_STRIDE); }
__global__ void k_t2_commit(Dev D, Cand C, T2Items T, Scr SC) {
  Scratch S = scratch_for(SC, GRID_START);
  t2_commit_body(D, C, T, S, GRID_START, GRID_STRIDE);
}
__global__ void k_t2_reset(Dev D, Cand C, T2Items T, int final_pass) { t2_reset_body(D, T, final_pass, GRID_START, GRID_STRIDE); }
__global__ void k_t2_retire(Dev D, T2Items T) { t2_retire_body(D, T, GRID_START, GRID_STRIDE); }
// every pass of a round in one block: no launches or host reads between passes
__global__ void __launch_bounds__(128) k_t2_fused(Dev D, Cand C, T2Items T, Scr SC, int* applied_total) {
  Scratch S = scratch_for(SC, threadIdx.x);
  __shared__ int s_applied;
  int left = T.n;
  for (int pass = 0; left > 0; ++pass) {
    if (threadIdx.x == 0) s_applied = 0;
    t2_compute_body(D, C, T, S, threadIdx.x, blockDim.x);
    __syncthreads();
    t2_claim_body(D, C, T, threadIdx.x, blockDim.x);
    __syncthreads();
    t2_apply_body(D, C, T, &s_applied, threadIdx.x, blockDim.x);
    __syncthreads();
    t2_reset_body(D, T, 1, threadIdx.x, blockDim.x);
    __syncthreads();
    t2_commit_body(D, C, T, S, threadIdx.x, blockDim.x);
    __syncthreads();
    t2_retire_body(D, T, threadIdx.x, blockDim.x);
    __syncthreads();
    const int applied = s_applied;
    __syncthreads();
    if (applied == 0) { if (threadIdx.x == 0) raise_err(GQ_ERR_2D); break; }
    left -= applied;
  }
  if (threadIdx.x == 0) *applied_total = T.n - left;
}

__global__ void k_kill_cavities(Dev D, Cand C, Ins I) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < I.n; k += gridDim.x * blockDim.x) {
    int c = I.list[k];
    SlabView v = slab(C, c);
    for (int j = 0; j < C.ntet[c]; ++j) D.alive[v.tets[j]] = 0;
  }
}
__global__ void k_star(Dev D, Cand C, Ins I) {
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
__global__ void __launch_bounds__(32 * WS_WARPS) k_star_warp(Dev D, Cand C, Ins I, Scr SB) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StarShared& X = reinterpret_cast<StarShared*>(smem_raw)[wib];
  const int gw = blockIdx.x * WS_WARPS + wib, nw = gridDim.x * WS_WARPS;
  for (int k = gw; k < I.n; k += nw) {
    int c = I.list[k];
    SlabView v = slab(C, c);
    int nbf = C.nbf[c];
    if (nbf <= WS_MAXF) star_warp(D, C.vid[c], v.bf, nbf, C.nt0[c], true, star_hash_shared(X), nullptr, 0);
    else star_warp(D, C.vid[c], v.bf, nbf, C.nt0[c], true, big_star_hash(SB, gw, &X.flag), nullptr, 0);
    __syncwarp();
  }
}
__global__ void __launch_bounds__(32 * WS_WARPS) k_init_stars_warp(Dev D, Cand C, const int* pend, const int* plist,
                                                                   const int* acc, int nw_, int* touched, int round, Scr SB) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StarShared& X = reinterpret_cast<StarShared*>(smem_raw)[wib];
  const int gw = blockIdx.x * WS_WARPS + wib, nw = gridDim.x * WS_WARPS;
  for (int w = gw; w < nw_; w += nw) {
    if (!acc[w]) continue;
    int c = plist[w];
    SlabView v = slab(C, c);
    int nbf = C.nbf[c];
    if (nbf <= WS_MAXF) star_warp(D, pend[c], v.bf, nbf, C.nt0[c], true, star_hash_shared(X), touched, round);
    else star_warp(D, pend[c], v.bf, nbf, C.nt0[c], true, big_star_hash(SB, gw, &X.flag), touched, round);
    __syncwarp();
    if (lane == 0) C.status[c] = CS_DROP;
  }
}

// dirty constraints + survivor mask refresh for subfaces retiled in 2D but
// not crossed by the 3D cavity (refine.py:720-736)
__global__ void k_post_insert(Dev D, Cand C, Ins I, T2Items T, Scr SC, const int* item_of) {
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

// ---------------------------------------------------------------------------
// constraint verification (refine.py:549-571, 829-851), mesh-local:
// a subsegment is tested against the vertices of the tets around it, a
// subface against the apexes of its two tets (identical to the
// reference's global KD-tree scans).
__device__ __noinline__ bool seg_check(const Dev& D, int r, Scratch& S) {   // true -> encroached or missing
  int2 e = D.sg_uv[r];
  const double *pu = PT(D, e.x), *pv = PT(D, e.y);
  bool present = false, enc = false;
  around_vertex(D, e.x, S.tset, S.stack, 2 * S.cap, [&](int t) {
    int4 q = D.tv[t];
    if (!has_v(q, e.y)) return false;
    present = true;
    for (int k = 0; k < 4; ++k) {
      int w = tvk(q, k);
      if (w == GHOST || w == e.x || w == e.y) continue;
      if (encroaches_segment(pu, pv, PT(D, w))) { enc = true; return true; }
    }
    return false;
  });
  return !present || enc;
}
__device__ __noinline__ bool face_check(const Dev& D, int r, Scratch& S) {
  int4 f = D.sf_v[r];
  int slot = find_face(D, f.x, f.y, f.z, S.tset, S.stack, 2 * S.cap);
  if (slot < 0) return true;
  const double *a = PT(D, f.x), *b = PT(D, f.y), *c = PT(D, f.z);
  int t = slot >> 2, i = slot & 3;
  int w = tvk(D.tv[t], i);
  if (w != GHOST && encroaches_face(a, b, c, PT(D, w))) return true;
  int nb = tnk(D, t, i);
  int u = nb >> 2, j = nb & 3;
  int w2 = tvk(D.tv[u], j);
  if (w2 != GHOST && encroaches_face(a, b, c, PT(D, w2))) return true;
  return false;
}
// mode 0: records flagged CHECK; mode 1: every live record (full_verify)
__global__ void k_check(Dev D, Scr SC, int mode, int* found) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  int ns = D.ctr->nsegrec, nf = D.ctr->nfacerec;
  for (int w = tid; w < ns + nf; w += gridDim.x * blockDim.x) {
    bool isseg = w < ns;
    int r = isseg ? w : w - ns;
    unsigned int* fl = isseg ? D.sg_fl + r : D.sf_fl + r;
    unsigned int f = *fl;
    if (!(f & RF_LIVE)) continue;
    if (mode == 0 && !(f & RF_CHECK)) continue;
    if (f & RF_CHECK) *fl = (f &= ~RF_CHECK);
    if ((f & RF_SKIP) || (f & RF_ENC)) continue;
    bool bad = isseg ? seg_check(D, r, S) : face_check(D, r, S);
    if (bad) { atomicOr(fl, RF_ENC); atomicAdd(found, 1); }
  }
}
__global__ void k_clear_flag(Dev D, unsigned int flag) {
  int ns = D.ctr->nsegrec, nf = D.ctr->nfacerec;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < ns + nf; w += gridDim.x * blockDim.x) {
    if (w < ns) D.sg_fl[w] &= ~flag; else D.sf_fl[w - ns] &= ~flag;
  }
}
// counts: [0] pending segs, [1] pending faces, [2] enc segs (live), [3] enc faces
__global__ void k_count_pending(Dev D, int* out) {
  int ns = D.ctr->nsegrec, nf = D.ctr->nfacerec;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < ns + nf; w += gridDim.x * blockDim.x) {
    unsigned int f = w < ns ? D.sg_fl[w] : D.sf_fl[w - ns];
    if (!(f & RF_LIVE) || !(f & RF_ENC)) continue;
    int base = w < ns ? 0 : 1;
    atomicAdd(out + 2 + base, 1);
    if (!(f & RF_BLOCK) && !(f & RF_SKIP)) atomicAdd(out + base, 1);
  }
}
__global__ void k_flag_pending_keys(Dev D, int phase, unsigned int need, unsigned int deny, int* flags,
                                    unsigned long long* k1, unsigned int* k2) {
  int ns = D.ctr->nsegrec, nf = D.ctr->nfacerec;
  int n = phase == 0 ? ns : nf;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    unsigned int f = phase == 0 ? D.sg_fl[r] : D.sf_fl[r];
    bool take = (f & RF_LIVE) && ((f & need) == need) && !(f & deny);
    flags[r] = take;
    if (phase == 0) { int2 e = D.sg_uv[r]; k1[r] = key2(e.x, e.y); }
    else { int4 q = D.sf_v[r]; k1[r] = key2(q.y, q.z); k2[r] = (unsigned int)q.x; }
  }
}
__global__ void k_face_a(Dev D, const int* recs, int n, unsigned int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = (unsigned int)D.sf_v[recs[i]].x;
}
__global__ void k_flag_bad(Dev D, double B, int* flags) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x)
    flags[t] = D.alive[t] == 1 && D.tv[t].w >= 0 && D.ratio[t] > B && D.skip[t] == 0;
}
__global__ void k_set_cands(Cand C, int n0, int n, int kind, const int* tgts, int pool0) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    C.kind[n0 + k] = kind; C.tgt[n0 + k] = tgts[k]; C.pool[n0 + k] = pool0 + k;
    C.status[n0 + k] = CS_OK; C.bigi[n0 + k] = -1;
  }
}
__global__ void k_clear_redir(Dev D, int phase) {
  int n = phase == 0 ? D.ctr->nsegrec : D.ctr->nfacerec;
  unsigned int* fl = phase == 0 ? D.sg_fl : D.sf_fl;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) fl[r] &= ~RF_REDIR;
}

// ---------------------------------------------------------------------------
// bulk Delaunay construction (mesh.py:869-943) as priority rounds: every
// pending point in a prefix window of the insertion order computes its
// cavity; the filter accepts points whose claims avoid every lower-order
// pending point, which makes the result the sequential one.
__global__ void k_init_first(Dev D, const int* order, int n, int* first_out) {
  if (blockIdx.x || threadIdx.x) return;
  int first[4]; int nf = 0;
  first[nf++] = order[0];
  for (int k = 1; k < n && nf < 4; ++k) {
    int idx = order[k];
    bool ok;
    if (nf == 1) {
      const double *a = PT(D, first[0]), *b = PT(D, idx);
      ok = !(a[0] == b[0] && a[1] == b[1] && a[2] == b[2]);
    } else if (nf == 2) {
      ok = false;
      for (int axis = 0; axis < 3 && !ok; ++axis) {
        int i = axis == 0 ? 1 : 0, j = axis == 2 ? 1 : 2;
        double a2[2] = {PT(D, first[0])[i], PT(D, first[0])[j]}, b2[2] = {PT(D, first[1])[i], PT(D, first[1])[j]};
        double c2[2] = {PT(D, idx)[i], PT(D, idx)[j]};
        if (orient2d(a2, b2, c2) != 0) ok = true;
      }
    } else {
      ok = orient3d(PT(D, first[0]), PT(D, first[1]), PT(D, first[2]), PT(D, idx)) != 0;
    }
    if (ok) first[nf++] = idx;
  }
  if (nf < 4) { raise_err(GQ_ERR_DEGEN); return; }
  int a = first[0], b = first[1], c = first[2], d = first[3];
  if (orient3d(PT(D, a), PT(D, b), PT(D, c), PT(D, d)) < 0) { int t = a; a = b; b = t; }
  D.tv[0] = make_int4(a, b, c, d);
  D.tn[0] = make_int4(-1, -1, -1, -1);
  D.alive[0] = 1; D.sub[0] = 0; D.seg[0] = 0; D.skip[0] = 0;
  for (int i = 0; i < 4; ++i) {
    int f[3]; face_verts(D.tv[0], i, f);
    int g = 1 + i;
    D.tv[g] = make_int4(f[0], f[1], f[2], GHOST);
    D.tn[g] = make_int4(-1, -1, -1, -1);
    D.alive[g] = 1; D.sub[g] = 0; D.seg[g] = 0; D.skip[g] = 0;
    set_tn(D, 0, i, 4 * g + 3);
    set_tn(D, g, 3, 4 * 0 + i);
  }
  for (int g = 1; g <= 4; ++g)
    for (int i = 0; i < 3; ++i) {
      if (tnk(D, g, i) >= 0) continue;
      int f[3]; face_verts(D.tv[g], i, f); sort3(f[0], f[1], f[2]);
      for (int g2 = g + 1; g2 <= 4; ++g2)
        for (int i2 = 0; i2 < 3; ++i2) {
          if (tnk(D, g2, i2) >= 0) continue;
          int h[3]; face_verts(D.tv[g2], i2, h); sort3(h[0], h[1], h[2]);
          if (h[0] == f[0] && h[1] == f[1] && h[2] == f[2]) { set_tn(D, g, i, 4 * g2 + i2); set_tn(D, g2, i2, 4 * g + i); }
        }
    }
  for (int t = 0; t < 5; ++t) {
    int4 q = D.tv[t];
    for (int k = 0; k < 4; ++k) { int v = tvk(q, k); if (v != GHOST) D.vert_tet[v] = t; }
  }
  star_ratio(D, 0);
  D.ratio[1] = D.ratio[2] = D.ratio[3] = D.ratio[4] = -1.0;
  D.ctr->nt = 5;
  for (int k = 0; k < 4; ++k) first_out[k] = first[k];
}

// Candidate c == pending point c (its position in the insertion order after
// the first tet).  A point's cavity stays cached across rounds while all its
// tets are alive and none of them was rewired since it was computed.
__global__ void k_init_region(Dev D, Cand C, Scr SC, const int* pend, const int* plist, int W, int* hint,
                              const int* succ, const int* touched, int round, int big) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  for (int w = tid; w < W; w += gridDim.x * blockDim.x) {
    int c = plist[w];
    int st = C.status[c];
    if (big) { if (st != CS_OVF || C.bigi[c] < 0) continue; }
    else if (st == CS_OK && C.memb[c] >= 0) {
      // cached: valid unless a cavity tet died or was rewired after round memb[c]
      SlabView v = slab(C, c);
      bool ok = true;
      for (int k = 0; k < C.ntet[c] && ok; ++k) {
        int t = v.tets[k];
        if (!D.alive[t] || touched[t] >= C.memb[c]) ok = false;   // rewired at/after computation
      }
      if (ok) continue;
    } else if (st == CS_OVF) continue;   // waits for the big pass
    int v = pend[c];
    const double* p = PT(D, v);
    int h = hint[c];
    if (h < 0) h = 0;
    while (h >= 0 && !D.alive[h]) h = succ[h];
    int t = walk(D, p, h);
    hint[c] = t;
    SlabView sv = slab(C, c);
    RegionOut O = region_view(C, c, sv, 0);
    int seeds[1] = {t};
    Allow A; A.n = 0;
    atomicAdd(&g_region_calls, 1ull);
    int r = region_compute(D, p, seeds, 1, A, S, O, true);
    store_region(C, c, O);
    C.extra[c] = -1; C.kind[c] = K_TET; C.rank[c] = c; C.memb[c] = round;
    if (r == RS_OK) { C.status[c] = CS_OK; atomicAdd(&g_tested, (unsigned long long)(O.ntet + O.nbf)); }
    else if (r == RS_OVERFLOW) { C.status[c] = CS_OVF; C.memb[c] = -1; if (big) raise_err(GQ_ERR_CAP); }
    else { C.status[c] = CS_CNSS; raise_err(GQ_ERR_DEGEN); }
  }
}
// window filter: claims of every window point, strict lower-order rule
__global__ void k_init_claim(Dev D, Cand C, Owners W, const int* plist, int nw) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    int c = plist[w];
    for_claims(D, C, W, c, [&](int k) { atomicMin(W.own + k, c); });
  }
}
__global__ void k_init_decide(Dev D, Cand C, Owners W, const int* plist, int nw, int* acc) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    int c = plist[w];
    bool win = true;
    for_claims(D, C, W, c, [&](int k) { if (W.own[k] != c) win = false; });
    acc[w] = win ? 1 : 0;
  }
}
__global__ void k_init_unclaim(Dev D, Cand C, Owners W, const int* plist, int nw) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    for_claims(D, C, W, plist[w], [&](int k) { W.own[k] = INT_MAX; });
}
// The window filter, tet-id assignment and cavity removal of one bulk round as
// one cooperative kernel: a warp per window point walks its claims
// lane-parallel; block 0 scans acceptance and boundary-face counts between the
// barriers; totals go to tot[0] (accepted) and tot[1] (new tets).
__global__ void __launch_bounds__(256) k_init_filter_coop(Dev D, Cand C, Owners W, const int* plist, int nw, int nt,
                                                          int* acc, int* accscan, int* nbfscan, int* tot, int* succ) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  const unsigned FULL = 0xffffffffu;
  for (int w = gw; w < nw; w += nwarp) {                    // claim: lowest order wins
    const int c = plist[w];
    warp_claims(D, C, W, c, lane, [&](int k) { atomicMin(W.own + k, c); });
  }
  grid.sync();
  for (int w = gw; w < nw; w += nwarp) {                    // decide
    const int c = plist[w];
    bool win = true;
    warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] != c) win = false; });
    win = __all_sync(FULL, win);
    if (lane == 0) acc[w] = win;
  }
  grid.sync();
  for (int w = gw; w < nw; w += nwarp)                      // release
    warp_claims(D, C, W, plist[w], lane, [&](int k) { W.own[k] = INT_MAX; });
  if (blockIdx.x == 0) {                                    // scans in insertion order
    typedef cub::BlockScan<int, 256> BS;
    __shared__ typename BS::TempStorage ts;
    __shared__ int carry[2];
    if (threadIdx.x == 0) carry[0] = carry[1] = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nw; b0 += 256) {
      const int w = b0 + threadIdx.x;
      const int a = w < nw ? acc[w] : 0;
      const int f = a ? C.nbf[plist[w]] : 0;
      int sa, sf, ta, tf;
      BS(ts).ExclusiveSum(a, sa, ta);
      __syncthreads();
      BS(ts).ExclusiveSum(f, sf, tf);
      if (w < nw) { accscan[w] = carry[0] + sa; nbfscan[w] = carry[1] + sf; }
      __syncthreads();
      if (threadIdx.x == 0) { carry[0] += ta; carry[1] += tf; }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      tot[0] = carry[0]; tot[1] = carry[1];
      if (nt + carry[1] > D.tcap) raise_err(GQ_ERR_CAP);
    }
  }
  grid.sync();
  for (int w = gw; w < nw; w += nwarp) {                    // new tet ids, cavities die
    if (!acc[w]) continue;
    const int c = plist[w];
    const int nt0 = nt + nbfscan[w];
    if (nt0 + C.nbf[c] > D.tcap) continue;
    if (lane == 0) {
      C.nt0[c] = nt0;
      if (C.mind[c] <= D.too_close_sq) raise_err(GQ_ERR_DEGEN);
    }
    SlabView v = slab(C, c);
    for (int j = lane; j < C.ntet[c]; j += 32) { D.alive[v.tets[j]] = 0; succ[v.tets[j]] = nt0; }
  }
}
// pending list minus the accepted window points (order kept)
__global__ void k_init_compact2(const int* plist, const int* acc, const int* accscan, int nw, int ntot, int nacc, int* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < ntot; w += gridDim.x * blockDim.x) {
    if (w < nw && acc[w]) continue;
    out[w < nw ? w - accscan[w] : w - nacc] = plist[w];
  }
}
// accepted window points: new tet ids (scan of nbf in insertion order)
__global__ void k_init_nbf(Cand C, const int* plist, const int* acc, int nw, int* nbfv) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    nbfv[w] = acc[w] ? C.nbf[plist[w]] : 0;
}
__global__ void k_init_kill(Dev D, Cand C, const int* plist, const int* acc, const int* scan, int nw, int nt,
                            int* succ) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    if (!acc[w]) continue;
    int c = plist[w];
    int nt0 = nt + scan[w];
    C.nt0[c] = nt0;
    if (C.mind[c] <= D.too_close_sq) raise_err(GQ_ERR_DEGEN);
    SlabView v = slab(C, c);
    for (int j = 0; j < C.ntet[c]; ++j) { D.alive[v.tets[j]] = 0; succ[v.tets[j]] = nt0; }
  }
}
__global__ void k_init_stars(Dev D, Cand C, const int* pend, const int* plist, const int* acc, int nw,
                             int* touched, int round) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    if (!acc[w]) continue;
    int c = plist[w];
    SlabView v = slab(C, c);
    for (int k = 0; k < C.nbf[c]; ++k) {      // survivors get rewired
      int t = v.bf[k] >> 2, i = v.bf[k] & 3;
      touched[tnk(D, t, i) >> 2] = round;
    }
    star_insert(D, pend[c], v.bf, C.nbf[c], C.nt0[c], true);
    C.status[c] = CS_DROP;
  }
}
__global__ void k_count_ovf(const Cand C, const int* plist, int W, int* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x)
    if (C.status[plist[w]] == CS_OVF) atomicAdd(out, 1);
    else if (C.status[plist[w]] == CS_OK) atomicMax(out + 1, C.ntet[plist[w]]);
}
__global__ void k_gather_status(const Cand C, const int* plist, int W, int* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) out[w] = C.status[plist[w]];
}
__global__ void k_release_big(Cand C, const int* list, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int c = list[k];
    if (C.status[c] != CS_DROP) { C.status[c] = CS_OK; C.memb[c] = -2; }   // -2: was big, route to the block kernel
    C.bigi[c] = -1;
  }
}
// remove accepted points from the pending list (stable)
__global__ void k_init_compact(const int* plist, const int* acc, const int* keepscan, int nw, int ntot, int* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < ntot; w += gridDim.x * blockDim.x) {
    if (w < nw && acc[w]) continue;
    int pos = w < nw ? keepscan[w] : (keepscan[nw - 1] + (acc[nw - 1] ? 0 : 1)) + (w - nw);
    out[pos] = plist[w];
  }
}
__global__ void k_init_keep(const int* acc, int nw, int* keep) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) keep[w] = acc[w] ? 0 : 1;
}

// facet bootstrap: one thread per polygon (facets.py:57-90, 342-372)
__global__ void k_facets_init(Dev D, const int* poff, const int* pidx, int f, Scr SC, int* t2base) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  for (int pid = tid; pid < f; pid += gridDim.x * blockDim.x) {
    int o0 = poff[pid], o1 = poff[pid + 1];
    Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = -2;
    int base[3]; int nb = 0;
    int last = -1;
    for (int k = o0; k < o1; ++k) {
      int v = pidx[k];
      if (nb < 3) {
        bool ok = true;
        double pa[2], pb[2], pc[2];
        if (nb == 1) { X.pos(base[0], pa); X.pos(v, pb); ok = !(pa[0] == pb[0] && pa[1] == pb[1]); }
        else if (nb == 2) { X.pos(base[0], pa); X.pos(base[1], pb); X.pos(v, pc); ok = orient2d(pa, pb, pc) != 0; }
        if (ok) base[nb++] = v;
        if (nb == 3) {
          int a = base[0], b = base[1], c = base[2];
          X.pos(a, pa); X.pos(b, pb); X.pos(c, pc);
          if (orient2d(pa, pb, pc) < 0) { int t = a; a = b; b = t; }
          last = t2_add(D, a, b, c, pid);
          t2_add(D, b, a, GHOST, pid); t2_add(D, c, b, GHOST, pid); t2_add(D, a, c, GHOST, pid);
        }
      }
    }
    if (nb < 3) { raise_err(GQ_ERR_DEGEN); continue; }
    // remaining corners in order (pending list: those not in base)
    for (int k = o0; k < o1; ++k) {
      int v = pidx[k];
      if (v == base[0] || v == base[1] || v == base[2]) continue;
      Tri2Ctx Y = X; Y.vid = v; X.pos(v, Y.p);
      int seeds[1] = {last};
      int cav[64];
      int n = tri2_cavity(Y, nullptr, 0, seeds, 1, S.tset, cav, S.stack, 64);
      if (n <= 0) { raise_err(GQ_ERR_2D); break; }
      S.tset.clear();
      for (int a = 0; a < n; ++a) S.tset.put(cav[a], a);
      int lastadd = -1;
      tri2_apply(Y, cav, n, S.tset, [&](int, int, int) {}, [&](int, int, int, int t2) { lastadd = t2; });
      if (lastadd >= 0) last = lastadd;
    }
  }
}
__global__ void k_facets_records(Dev D, int nt2) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt2; t += gridDim.x * blockDim.x) {
    if (!D.t2alive[t]) continue;
    int4 q = D.t2v[t];
    if (q.z == GHOST) continue;
    new_face_record(D, q.x, q.y, q.z, q.w, RF_LIVE);
  }
}
__global__ void k_segs_init(Dev D, const int* seg, int m) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    int u = seg[2 * s], v = seg[2 * s + 1];
    if (u > v) { int t = u; u = v; v = t; }
    D.sg_uv[s] = make_int2(u, v); D.sg_sid[s] = s; D.sg_fl[s] = RF_LIVE;
    D.sid_uv[s] = make_int2(u, v);
    ht_put(D.sg_hk, D.sg_hv, D.sg_hmask, key2(u, v), s);
  }
}
__global__ void k_refresh_all(Dev D) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x)
    if (D.alive[t]) refresh_masks(D, t);
}

// ---------------------------------------------------------------------------
// sequential fallback for failed candidates (refine.py:748-799): one thread,
// in pool order, on the updated mesh.  Uses the big scratch / slab 0.
struct FallbackIO { const int* list; int n; int round_no; unsigned long long seed; int with_facets; double lmin2; int* inserted; };

__device__ inline void mark_enc_face_key(const Dev& D, int a, int b, int c) {
  sort3(a, b, c);
  int r = face_lookup(D, a, b, c);
  if (r >= 0 && !(D.sf_fl[r] & RF_SKIP)) D.sf_fl[r] |= RF_ENC;
}
__device__ __noinline__ void skip_cand(const Dev& D, const Cand& C, int c, int reason, int round_no, const SkipLog& L) {
  int kind = C.kind[c], tgt = C.tgt[c];
  if (kind == K_TET) {
    if (tgt >= 0 && tgt < D.ctr->nt && D.alive[tgt]) {
      D.skip[tgt] = 1;
      int cv[4]; tet_canon(D, tgt, cv);
      log_skip(D, L, round_no, K_TET, reason, cv, 4);
    }
  } else if (kind == K_SEG) {
    D.sg_fl[tgt] = (D.sg_fl[tgt] | RF_SKIP) & ~RF_ENC;
    int2 e = D.sg_uv[tgt]; int v[2] = {e.x, e.y};
    log_skip(D, L, round_no, K_SEG, reason, v, 2);
  } else {
    D.sf_fl[tgt] = (D.sf_fl[tgt] | RF_SKIP) & ~RF_ENC;
    int4 f = D.sf_v[tgt]; int v[3] = {f.x, f.y, f.z};
    log_skip(D, L, round_no, K_FACE, reason, v, 3);
  }
}

__device__ __noinline__ void insert_one(const Dev& D, const Cand& C, int c, Scratch& S, T2Items& T, int item0) {
  // sequential insert_candidate: vid, 2D retile per polygon, split, star
  int vid = atomicAdd(&D.ctr->nv, 1);
  C.vid[c] = vid;
  const double* p = C.p + 3 * (size_t)c;
  double* q = D.P + 3 * (size_t)vid;
  q[0] = p[0]; q[1] = p[1]; q[2] = p[2];
  D.vorigin[vid] = 1; D.vert_tet[vid] = -1;
  D.vsid[vid] = C.kind[c] == K_SEG ? D.sg_sid[C.tgt[c]] : -1;
  int nitems = 0;
  if (C.kind[c] != K_TET && D.npoly > 0) {
    int pids[8]; int np = 0;
    if (C.kind[c] == K_SEG) {
      int sid = D.sg_sid[C.tgt[c]];
      for (int o = D.segpoly_off[sid]; o < D.segpoly_off[sid + 1] && np < 8; ++o) pids[np++] = D.segpoly[o];
    } else pids[np++] = D.sf_v[C.tgt[c]].w;
    for (int k = 0; k < np; ++k) {
      int w = item0 + k;
      int pid = pids[k];
      Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = vid;
      proj2(D, pid, p, X.p);
      int forced[CC + 2]; int nf;
      t2_forced(D, C, c, pid, forced, nf, CC + 2);
      int seeds[CC + 3]; int ns = 0;
      for (int j = 0; j < nf; ++j) seeds[ns++] = forced[j];
      int ts = t2_seed_of(D, C, c, pid);
      if (ts >= 0) seeds[ns++] = ts;
      int* cav = T.cav + (size_t)w * T.cap;
      int n = tri2_cavity(X, forced, nf, seeds, ns, S.tset, cav, S.stack, T.cap);
      if (n < 0) {
#ifdef GQ_DEBUG2D
      printf("[2d] cavity fail pid %d vid %d\n", pid, X.vid);
#endif
      raise_err(GQ_ERR_2D); n = 0;
    }
      S.tset.clear();
      for (int a = 0; a < n; ++a) S.tset.put(cav[a], a);
      int* rem = T.rem + (size_t)w * T.rcap;
      int nrem = 0;
      tri2_apply(X, cav, n, S.tset,
        [&](int a, int b, int cc) {
          sort3(a, b, cc);
          int rec = face_lookup(D, a, b, cc);
          if (rec >= 0 && D.sf_v[rec].w == pid) { if (nrem < T.rcap) rem[nrem++] = rec; }
        },
        [&](int a, int b, int cc, int) {
          if (collinear_sliver(D, a, b, cc)) return;
          int a0 = a, b0 = b, c0 = cc; sort3(a0, b0, c0);
          if (face_lookup(D, a0, b0, c0) >= 0) return;
          new_face_record(D, a0, b0, c0, pid, RF_LIVE | RF_CHECK);
        });
      T.nrem[w] = nrem;
      for (int j = 0; j < nrem; ++j) D.sf_fl[rem[j]] = 0;
      ++nitems;
    }
  }
  if (C.kind[c] == K_SEG) {
    int r = C.tgt[c];
    int2 e = D.sg_uv[r];
    int sid = D.sg_sid[r];
    D.sg_fl[r] = 0;
    new_seg_record(D, e.x, vid, sid, RF_LIVE | RF_CHECK);
    new_seg_record(D, e.y, vid, sid, RF_LIVE | RF_CHECK);
  }
  SlabView v = slab(C, c);
  for (int j = 0; j < C.ntet[c]; ++j) D.alive[v.tets[j]] = 0;
  int nt0 = atomicAdd(&D.ctr->nt, C.nbf[c]);
  if (nt0 + C.nbf[c] > D.tcap) { raise_err(GQ_ERR_CAP); return; }
  C.nt0[c] = nt0;
  star_insert(D, vid, v.bf, C.nbf[c], nt0, false);
  for (int j = 0; j < C.nbsub[c]; ++j) { int r = v.bsub[j]; if (r >= 0 && (D.sf_fl[r] & RF_LIVE)) D.sf_fl[r] |= RF_CHECK; }
  for (int j = 0; j < C.nbseg[c]; ++j) { int r = v.bseg[j]; if (r >= 0 && (D.sg_fl[r] & RF_LIVE)) D.sg_fl[r] |= RF_CHECK; }
  for (int w = item0; w < item0 + nitems; ++w) {
    const int* rem = T.rem + (size_t)w * T.rcap;
    for (int j = 0; j < T.nrem[w]; ++j) {
      int rec = rem[j];
      bool crossed = false;
      for (int qq = 0; qq < C.ncr[c]; ++qq) if (v.cr[qq] == rec) { crossed = true; break; }
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

__global__ void k_fallback(Dev D, Cand C, Scr SCB, FallbackIO F, T2Items T, SkipLog L) {
  if (blockIdx.x || threadIdx.x) return;
  Scratch S = scratch_for(SCB, 0);
  CandCtx X; X.round_no = F.round_no; X.seed = F.seed; X.with_facets = F.with_facets;
  for (int k = 0; k < F.n; ++k) {
    int c = F.list[k];
    int kind = C.kind[c], tgt = C.tgt[c];
    if (C.status[c] == CS_TOOCLOSE) { skip_cand(D, C, c, 2, F.round_no, L); continue; }
    if (kind == K_TET && !(tgt >= 0 && tgt < D.ctr->nt && D.alive[tgt])) continue;
    if (kind == K_SEG && !(D.sg_fl[tgt] & RF_LIVE)) continue;
    if (kind == K_FACE && !(D.sf_fl[tgt] & RF_LIVE)) continue;
    if (!make_cand(D, C, c, X, S)) { raise_err(GQ_ERR_DEGEN); continue; }
    const double* p = C.p + 3 * (size_t)c;
    if (kind == K_TET) {
      int cur = tgt, prev = -1, hull = -2;
      int max_steps = walk_cap(D, 64);
      bool done = false;
      for (int step = 0; step < max_steps && !done; ++step) {
        int4 q = D.tv[cur];
        if (q.w == GHOST) { int a = q.x, b = q.y, cc = q.z; sort3(a, b, cc); hull = face_lookup(D, a, b, cc); if (hull < 0) hull = -1; done = true; break; }
        bool moved = false;
        for (int kk = 0; kk < 4; ++kk) {
          int i = (kk + step) & 3;
          int u = tnk(D, cur, i) >> 2;
          if (u == prev) continue;
          int f[3]; face_verts(q, i, f);
          if (orient3d(PT(D, f[0]), PT(D, f[1]), PT(D, f[2]), p) > 0) {
            if (D.tv[u].w == GHOST) { sort3(f[0], f[1], f[2]); hull = face_lookup(D, f[0], f[1], f[2]); if (hull < 0) hull = -1; done = true; break; }
            prev = cur; cur = u; moved = true; break;
          }
        }
        if (done) break;
        if (!moved) { done = true; break; }
      }
      if (!done) {
        int end = walk(D, p, tgt);
        if (end >= 0 && D.tv[end].w == GHOST) { int4 q = D.tv[end]; int a = q.x, b = q.y, cc = q.z; sort3(a, b, cc); hull = face_lookup(D, a, b, cc); if (hull < 0) hull = -1; }
      }
      if (hull >= 0) {   // redirect the subface to the next round
        if (!(D.sf_fl[hull] & RF_SKIP)) D.sf_fl[hull] |= RF_ENC;
        continue;
      }
    }
    C.bigi[c] = 0;
    SlabView sv = slab(C, c);
    RegionOut O = region_view(C, c, sv, 0);
    int seeds[32];
    int ns = cand_seeds(D, C, c, seeds, S);
    atomicAdd(&g_region_calls, 1ull);
    int st = ns == 0 ? RS_CNSS : region_compute(D, p, seeds, ns, allow_of(C, c), S, O);
    store_region(C, c, O);
    if (st == RS_OK) {
      if (O.mind <= D.too_close_sq) { skip_cand(D, C, c, 2, F.round_no, L); continue; }
      if (kind == K_TET && O.mind < F.lmin2) {
        D.skip[tgt] = 1;
        int cv[4]; tet_canon(D, tgt, cv);
        log_skip(D, L, F.round_no, K_TET, 1, cv, 4);
        continue;
      }
      if (D.ctr->nv >= D.vcap) { raise_err(GQ_ERR_CAP); return; }
      insert_one(D, C, c, S, T, 0);
      atomicAdd(F.inserted, 1);
    } else if (st == RS_MEMBRANE) {
      int t = O.memb >> 2, i = O.memb & 3;
      int f[3]; face_verts(D.tv[t], i, f);
      mark_enc_face_key(D, f[0], f[1], f[2]);
      if (kind == K_SEG) D.sg_fl[tgt] |= RF_BLOCK;
      else if (kind == K_FACE) D.sf_fl[tgt] |= RF_BLOCK;
    } else {
      if (st == RS_OVERFLOW) raise_err(GQ_ERR_CAP);
      skip_cand(D, C, c, 3, F.round_no, L);
    }
  }
}

// accepted tets whose region has a too-short boundary edge (refine.py:891-894)
__global__ void k_accept_flags(Dev D, Cand C, const int* acc, int nacc, int* insflag, SkipLog L, int round_no, double lmin2) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nacc; k += gridDim.x * blockDim.x) {
    int c = acc[k];
    if (C.kind[c] == K_TET && C.mind[c] < lmin2) {
      insflag[k] = 0;
      int t = C.tgt[c];
      if (t >= 0 && D.alive[t]) {
        D.skip[t] = 1;
        int cv[4]; tet_canon(D, t, cv);
        log_skip(D, L, round_no, K_TET, 1, cv, 4);
      }
    } else insflag[k] = 1;
  }
}
__global__ void k_assign_ids(Cand C, const int* ins, int n, const int* nbfscan, int nv0, int nt0) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int c = ins[k];
    C.vid[c] = nv0 + k;
    C.nt0[c] = nt0 + nbfscan[k];
  }
}
__global__ void k_gather_nbf(Cand C, const int* ins, int n, int* out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = C.nbf[ins[k]];
}
__global__ void k_rank_scatter(Cand C, const int* order, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) C.rank[order[k]] = k;
}

// compaction of dead tet slots (mesh.py:847-865), stable
__global__ void k_compact_flags(Dev D, int* flags) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) flags[t] = D.alive[t] == 1;
}
__global__ void k_compact_move(Dev D, const int* remap, int nt, int4* tv2, int4* tn2, uint8_t* sub2, uint8_t* seg2,
                               double* ratio2, uint8_t* skip2) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    if (D.alive[t] != 1) continue;
    int r = remap[t];
    tv2[r] = D.tv[t];
    int4 q = D.tn[t];
    tn2[r] = make_int4(remap[q.x >> 2] * 4 + (q.x & 3), remap[q.y >> 2] * 4 + (q.y & 3),
                       remap[q.z >> 2] * 4 + (q.z & 3), remap[q.w >> 2] * 4 + (q.w & 3));
    sub2[r] = D.sub[t]; seg2[r] = D.seg[t]; ratio2[r] = D.ratio[t]; skip2[r] = D.skip[t];
  }
}
__global__ void k_compact_vt(Dev D, const int* remap, const int* flags, int nv) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int t = D.vert_tet[v];
    D.vert_tet[v] = t >= 0 ? (flags[t] ? remap[t] : -1) : -1;
  }
}

// quality (stats.py:35-99): bad count + dihedral histogram of real tets
__global__ void k_quality(Dev D, double B, unsigned long long* bad, unsigned long long* hist) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    if (!D.alive[t] || D.tv[t].w == GHOST) continue;
    int4 q = D.tv[t];
    const double* P4[4] = {PT(D, q.x), PT(D, q.y), PT(D, q.z), PT(D, q.w)};
    double a[3], u[3], v[3], w[3];
    for (int k = 0; k < 3; ++k) { a[k] = P4[0][k]; u[k] = P4[1][k] - a[k]; v[k] = P4[2][k] - a[k]; w[k] = P4[3][k] - a[k]; }
    double vw[3] = {v[1] * w[2] - v[2] * w[1], v[2] * w[0] - v[0] * w[2], v[0] * w[1] - v[1] * w[0]};
    double wu[3] = {w[1] * u[2] - w[2] * u[1], w[2] * u[0] - w[0] * u[2], w[0] * u[1] - w[1] * u[0]};
    double uv[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    double denom = 2.0 * (u[0] * vw[0] + u[1] * vw[1] + u[2] * vw[2]);
    double lu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    double lv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    double lw = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    double off[3];
    for (int k = 0; k < 3; ++k) off[k] = (lu * vw[k] + lv * wu[k] + lw * uv[k]) / denom;
    double r2 = off[0] * off[0] + off[1] * off[1] + off[2] * off[2];
    double sh = INFINITY;
    const int pr[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    for (int e = 0; e < 6; ++e) {
      double d = dist2(P4[pr[e][0]], P4[pr[e][1]]);
      sh = d < sh ? d : sh;
    }
    double ratio = sqrt(r2 / sh);
    if (!isfinite(ratio)) ratio = INFINITY;
    if (ratio > B) atomicAdd(bad, 1ull);
    for (int e = 0; e < 6; ++e) {
      int i = pr[e][0], j = pr[e][1];
      int kk = -1, ll = -1;
      for (int m = 0; m < 4; ++m) if (m != i && m != j) { if (kk < 0) kk = m; else ll = m; }
      double ed[3], ek[3], el[3];
      for (int k = 0; k < 3; ++k) { ed[k] = P4[j][k] - P4[i][k]; ek[k] = P4[kk][k] - P4[i][k]; el[k] = P4[ll][k] - P4[i][k]; }
      double n1[3] = {ed[1] * ek[2] - ed[2] * ek[1], ed[2] * ek[0] - ed[0] * ek[2], ed[0] * ek[1] - ed[1] * ek[0]};
      double n2[3] = {ed[1] * el[2] - ed[2] * el[1], ed[2] * el[0] - ed[0] * el[2], ed[0] * el[1] - ed[1] * el[0]};
      double dot = n1[0] * n2[0] + n1[1] * n2[1] + n1[2] * n2[2];
      double nrm = sqrt((n1[0] * n1[0] + n1[1] * n1[1] + n1[2] * n1[2]) * (n2[0] * n2[0] + n2[1] * n2[1] + n2[2] * n2[2]));
      double ca = dot / nrm;
      ca = ca < -1.0 ? -1.0 : (ca > 1.0 ? 1.0 : ca);
      double ang = acos(ca) * (180.0 / 3.14159265358979323846);
      int bin = (int)(ang / 5.0);
      bin = bin < 0 ? 0 : (bin > 35 ? 35 : bin);
      if (!(ang == ang)) bin = 0;
      atomicAdd(hist + bin, 1ull);
    }
  }
}

// batched predicates / constructions for parity tests (gq_batch)
__global__ void k_batch(int which, const double* in, int n, signed char* out8, double* outd) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* x;
    switch (which) {
      case 0: x = in + 12 * (size_t)i; out8[i] = (signed char)orient3d(x, x + 3, x + 6, x + 9); break;
      case 1: x = in + 15 * (size_t)i; out8[i] = (signed char)insphere(x, x + 3, x + 6, x + 9, x + 12); break;
      case 2: x = in + 6 * (size_t)i; out8[i] = (signed char)orient2d(x, x + 2, x + 4); break;
      case 3: x = in + 8 * (size_t)i; out8[i] = (signed char)incircle2d(x, x + 2, x + 4, x + 6); break;
      case 4: {
        x = in + 12 * (size_t)i;
        unsigned int before = g_err;
        int r = incircle3d(x, x + 3, x + 6, x + 9);
        // degenerate triangle: the reference raises; report 99
        double ux = x[3] - x[0], uy = x[4] - x[1], uz = x[5] - x[2], vx = x[6] - x[0], vy = x[7] - x[1], vz = x[8] - x[2];
        double a2[2], b2[2], c2[2]; bool deg = true;
        for (int axis = 0; axis < 3 && deg; ++axis) {
          int p = axis == 0 ? 1 : 0, q = axis == 2 ? 1 : 2;
          a2[0] = x[p]; a2[1] = x[q]; b2[0] = x[3 + p]; b2[1] = x[3 + q]; c2[0] = x[6 + p]; c2[1] = x[6 + q];
          if (orient2d(a2, b2, c2) != 0) deg = false;
        }
        (void)before; (void)ux; (void)uy; (void)uz; (void)vx; (void)vy; (void)vz;
        out8[i] = deg ? 99 : (signed char)r;
        break;
      }
      case 5: x = in + 9 * (size_t)i; out8[i] = encroaches_segment(x, x + 3, x + 6) ? 1 : 0; break;
      case 6: {
        x = in + 12 * (size_t)i;
        Sphere sp;
        if (!circumcircle_tri(x, x + 3, x + 6, sp)) { out8[i] = 99; break; }
        out8[i] = encroaches_face(x, x + 3, x + 6, x + 9) ? 1 : 0;
        break;
      }
      case 7: {
        x = in + 12 * (size_t)i;
        Sphere sp;
        if (circumsphere_tet(x, x + 3, x + 6, x + 9, sp) != 0) { for (int k = 0; k < 4; ++k) outd[4 * (size_t)i + k] = nan(""); }
        else { outd[4 * (size_t)i] = sp.c[0]; outd[4 * (size_t)i + 1] = sp.c[1]; outd[4 * (size_t)i + 2] = sp.c[2]; outd[4 * (size_t)i + 3] = sp.r2; }
        break;
      }
      case 8: {
        x = in + 9 * (size_t)i;
        Sphere sp;
        if (!circumcircle_tri(x, x + 3, x + 6, sp)) { for (int k = 0; k < 4; ++k) outd[4 * (size_t)i + k] = nan(""); }
        else { outd[4 * (size_t)i] = sp.c[0]; outd[4 * (size_t)i + 1] = sp.c[1]; outd[4 * (size_t)i + 2] = sp.c[2]; outd[4 * (size_t)i + 3] = sp.r2; }
        break;
      }
    }
  }
}

// ===========================================================================
// host driver
// ===========================================================================

// Caching device allocator.  A refine allocates a few GB of mesh, candidate and
// scratch arrays; repeated refines on a context (bench steps, batches of PLCs)
// reuse them instead of paying cudaMalloc / cudaFree (a device-wide sync) in
// the middle of the rounds.  Blocks are binned in size classes (<= 25% slack);
// everything runs on the context's single stream, so reuse is stream-ordered.
struct DevCache {
  std::mutex mu;
  std::unordered_multimap<size_t, void*> free_blocks;
  std::unordered_map<void*, size_t> live;
};
static DevCache& dev_cache() {
  static DevCache caches[64];
  int d = 0;
  cudaGetDevice(&d);
  return caches[d & 63];
}
static size_t size_class(size_t b) {
  if (b <= 4096) return 4096;
  size_t p = 4096;
  while (p < b) p <<= 1;
  size_t step = p / 8;
  return (b + step - 1) / step * step;
}
static void cache_trim(DevCache& C) {
  for (auto& kv : C.free_blocks) cudaFree(kv.second);
  C.free_blocks.clear();
}
static void* cache_alloc(size_t bytes) {
  DevCache& C = dev_cache();
  std::lock_guard<std::mutex> g(C.mu);
  size_t cls = size_class(bytes);
  auto it = C.free_blocks.find(cls);
  void* p = nullptr;
  if (it != C.free_blocks.end()) {
    p = it->second;
    C.free_blocks.erase(it);
  } else if (cudaMalloc(&p, cls) != cudaSuccess) {
    cudaGetLastError();
    cache_trim(C);                       // out of memory: return the cached blocks, retry once
    CK(cudaMalloc(&p, cls));
  }
  C.live[p] = cls;
  return p;
}
static void dfree(void* p) {
  if (!p) return;
  DevCache& C = dev_cache();
  std::lock_guard<std::mutex> g(C.mu);
  auto it = C.live.find(p);
  if (it == C.live.end()) { cudaFree(p); return; }
  C.free_blocks.emplace(it->second, p);
  C.live.erase(it);
}
template <class T> static T* dmalloc(size_t n) {
  if (n == 0) n = 1;
  return (T*)cache_alloc(n * sizeof(T));
}

struct gq_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  Dev D{};
  Counters* dctr = nullptr;
  Counters hc{};
  Cand C{};
  Scr S{}, SB{};
  Owners W{};
  SkipLog L{};
  T2Items T{};
  int* d_int = nullptr;     // small int scratch (64)
  int* d_order = nullptr;
  // temp buffers
  int* tmpA = nullptr; int* tmpB = nullptr; int* tmpC = nullptr; size_t tmpcap = 0;
  unsigned long long* k64a = nullptr; unsigned long long* k64b = nullptr; unsigned int* k32a = nullptr; unsigned int* k32b = nullptr;
  void* cub_tmp = nullptr; size_t cub_cap = 0;
  // config / state
  double B = 2.0; int max_rounds = 500; unsigned long long seed = 0; bool verbose = false; bool blast = false;   // blast: paper-literal grow-and-blast filter (flags bit 1)
  int n_input = 0, npoly = 0;
  std::vector<std::array<long long, 9>> rounds;
  std::vector<double> rtimes;
  long long launches = 0;
  double init_ms = 0, dev_ms = 0, region_ms = 0;
  cudaEvent_t ev0, ev1, er0, er1;
  // event pool: region-kernel timing and the GQ_PROFILE=3 stage timeline are
  // resolved once at the end of a refine, never by a per-launch sync
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> rpairs;
  std::vector<std::pair<cudaEvent_t, int>> fev;
  std::vector<std::vector<int>> polys;
  CGrid G{};
  int reg_seg = 0, reg_face = 0, reg_nv = 0;
  int big_used = 0;
  int init_rounds = 0;
  long long grid_calls = 0;
  int4 *tv2 = nullptr, *tn2 = nullptr; uint8_t *sub2 = nullptr, *seg2 = nullptr, *skip2 = nullptr; double* ratio2 = nullptr;
  struct QBuf { int *a, *b, *c, *d, *e, *f, *g, *h; size_t cap; } Q{};
  bool allocated = false;
};

static double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static double g_prof[8];
// fine stage timers (GQ_PROFILE=2): synchronise and charge the elapsed time
static bool g_trace = false;
static bool g_fine = false;      // GQ_PROFILE=2: host clock after a sync per stage
static bool g_fine_ev = false;   // GQ_PROFILE=3: events per stage (device timeline, no syncs)
static double g_fine_t[32];
static const char* g_fine_names[32] = {"i.region", "i.big", "i.filter", "i.scan", "i.kill", "i.stars", "i.compact",
  "p.gridsync", "p.newverts", "p.check", "p.compact", "r.sorted", "r.make", "r.redirect", "r.append", "f.states",
  "f.rank", "f.lfmis", "x.acc", "x.ids", "x.star", "x.postins", "i.misc", "r.misc", "g.warp", "g.ovfscan", "g.block",
  "r.setup", "r.gridc", "r.kept", "x.fallback", "r.misc2"};
static double g_fine_last = 0;
static void fine(gq_ctx* c, int k);
static void sync(gq_ctx* c) {
  CK(cudaStreamSynchronize(c->st));
  unsigned int e = 0;
  CK(cudaMemcpyFromSymbol(&e, g_err, sizeof(e)));
  if (e) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "device error flags 0x%x", e);
    throw std::runtime_error(buf);
  }
}
static void pull(gq_ctx* c) { CK(cudaMemcpyAsync(&c->hc, c->dctr, sizeof(Counters), cudaMemcpyDeviceToHost, c->st)); sync(c); }
static void push(gq_ctx* c) { CK(cudaMemcpyAsync(c->dctr, &c->hc, sizeof(Counters), cudaMemcpyHostToDevice, c->st)); }
static int grid_for(long long n, int bs = 128, int cap = 148 * 16) {
  long long g = (n + bs - 1) / bs;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}
#define LAUNCH(kern, n, ...) do { kern<<<grid_for(n), 128, 0, c->st>>>(__VA_ARGS__); c->launches++; CK(cudaGetLastError()); } while (0)
#define LAUNCH_S(kern, n, ...) do { kern<<<grid_for(n, 128, c->S.nthreads / 128), 128, 0, c->st>>>(__VA_ARGS__); c->launches++; CK(cudaGetLastError()); } while (0)

static void ensure_cub(gq_ctx* c, size_t need) {
  if (need <= c->cub_cap) return;
  dfree(c->cub_tmp);
  c->cub_cap = need * 2;
  c->cub_tmp = dmalloc<char>(c->cub_cap);
}
static void ensure_tmp(gq_ctx* c, size_t n) {
  if (n <= c->tmpcap) return;
  for (void* p : {(void*)c->tmpA, (void*)c->tmpB, (void*)c->tmpC, (void*)c->k64a, (void*)c->k64b, (void*)c->k32a, (void*)c->k32b})
    if (p) dfree(p);
  c->tmpcap = n * 2;
  c->tmpA = dmalloc<int>(c->tmpcap); c->tmpB = dmalloc<int>(c->tmpcap); c->tmpC = dmalloc<int>(c->tmpcap);
  c->k64a = dmalloc<unsigned long long>(c->tmpcap); c->k64b = dmalloc<unsigned long long>(c->tmpcap);
  c->k32a = dmalloc<unsigned int>(c->tmpcap); c->k32b = dmalloc<unsigned int>(c->tmpcap);
}
__global__ void k_gather_u32(const unsigned int* src, const int* idx, int n, unsigned int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}
__global__ void k_gather_u64(const unsigned long long* src, const int* idx, int n, unsigned long long* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}
__global__ void k_scatter_ints(int* dst, const int* idx, const int* val, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[idx[i]] = val[i];
}
__global__ void k_scatter_flagged(const int* flags, const int* scan, int n, int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (flags[i]) out[scan[i]] = i;
}
static void exclusive_scan(gq_ctx* c, const int* in, int* out, int n);
// indices i in [0,n) with flags[i] != 0, in order -> out; returns count
static int select_flagged(gq_ctx* c, const int* flags, int n, int* out) {
  if (n <= 0) return 0;
  ensure_tmp(c, n + 1);
  exclusive_scan(c, flags, c->tmpC, n);
  LAUNCH(k_scatter_flagged, n, flags, c->tmpC, n, out);
  int last_f = 0, last_s = 0;
  CK(cudaMemcpyAsync(&last_f, flags + n - 1, 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(&last_s, c->tmpC + n - 1, 4, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return last_f + last_s;
}
static void exclusive_scan(gq_ctx* c, const int* in, int* out, int n) {
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n, c->st);
  ensure_cub(c, need);
  cub::DeviceScan::ExclusiveSum(c->cub_tmp, need, in, out, n, c->st);
}
static int read_int(gq_ctx* c, const int* d) { int v; CK(cudaMemcpyAsync(&v, d, sizeof v, cudaMemcpyDeviceToHost, c->st)); sync(c); return v; }

static void alloc_scratch(Scr& s, int nthreads, int cap, int tcap, int fcap) {
  s.nthreads = nthreads; s.cap = cap; s.tcap = tcap; s.fcap = fcap;
  s.tkey = dmalloc<int>((size_t)nthreads * tcap); s.tval = dmalloc<int>((size_t)nthreads * tcap);
  s.tep = dmalloc<unsigned int>((size_t)nthreads * tcap);
  s.fkey = dmalloc<unsigned long long>((size_t)nthreads * fcap); s.fep = dmalloc<unsigned int>((size_t)nthreads * fcap);
  s.epoch = dmalloc<unsigned int>((size_t)nthreads * 2);
  CK(cudaMemset(s.tep, 0, (size_t)nthreads * tcap * 4)); CK(cudaMemset(s.fep, 0, (size_t)nthreads * fcap * 4));
  CK(cudaMemset(s.epoch, 0, (size_t)nthreads * 2 * 4));
  s.list = dmalloc<int>((size_t)nthreads * cap); s.stack = dmalloc<int>((size_t)nthreads * cap * 2);
  s.in = dmalloc<uint8_t>((size_t)nthreads * cap); s.comp = dmalloc<uint8_t>((size_t)nthreads * cap);
}

static void alloc_cands(gq_ctx* c, int cap, int bigcap) {
  Cand& C = c->C;
  C.cap = cap;
  C.kind = dmalloc<int>(cap); C.tgt = dmalloc<int>(cap); C.seed = dmalloc<int>(cap); C.status = dmalloc<int>(cap);
  C.memb = dmalloc<int>(cap); C.pool = dmalloc<int>(cap); C.rank = dmalloc<int>(cap);
  C.allow = dmalloc<int4>(cap); C.nallow = dmalloc<int>(cap); C.extra = dmalloc<int>(cap);
  C.p = dmalloc<double>(3 * (size_t)cap); C.h = dmalloc<unsigned long long>(cap); C.canon = dmalloc<int4>(cap);
  C.state = dmalloc<int>(cap); C.vid = dmalloc<int>(cap); C.nt0 = dmalloc<int>(cap);
  C.ntet = dmalloc<int>(cap); C.nbf = dmalloc<int>(cap); C.ncr = dmalloc<int>(cap); C.nbsub = dmalloc<int>(cap);
  C.nbseg = dmalloc<int>(cap); C.neseg = dmalloc<int>(cap); C.mind = dmalloc<double>(cap);
  C.tets = dmalloc<int>((size_t)cap * CT); C.bf = dmalloc<int>((size_t)cap * CF);
  C.cr = dmalloc<int>((size_t)cap * CC); C.crf = dmalloc<int>((size_t)cap * CC); C.bsub = dmalloc<int>((size_t)cap * CC);
  C.bseg = dmalloc<int>((size_t)cap * CC); C.eseg = dmalloc<int>((size_t)cap * CC);
  C.rseg = dmalloc<int>((size_t)cap * CRD); C.rface = dmalloc<int>((size_t)cap * CRD);
  C.nrseg = dmalloc<int>(cap); C.nrface = dmalloc<int>(cap);
  C.bigi = dmalloc<int>(cap);
  C.nbigcap = bigcap;
  C.btets = dmalloc<int>((size_t)bigcap * CTB); C.bbf = dmalloc<int>((size_t)bigcap * CFB);
  C.bcr = dmalloc<int>((size_t)bigcap * CCB); C.bcrf = dmalloc<int>((size_t)bigcap * CCB);
  C.bbsub = dmalloc<int>((size_t)bigcap * CCB); C.bbseg = dmalloc<int>((size_t)bigcap * CCB);
  C.beseg = dmalloc<int>((size_t)bigcap * CCB);
}
static void free_cands(Cand& C) {
  void* ps[] = {C.kind, C.tgt, C.seed, C.status, C.memb, C.pool, C.rank, C.allow, C.nallow, C.extra, C.p, C.h, C.canon,
                C.state, C.vid, C.nt0, C.ntet, C.nbf, C.ncr, C.nbsub, C.nbseg, C.neseg, C.mind, C.tets, C.bf, C.cr,
                C.crf, C.bsub, C.bseg, C.eseg, C.rseg, C.rface, C.nrseg, C.nrface, C.bigi, C.btets, C.bbf, C.bcr,
                C.bcrf, C.bbsub, C.bbseg, C.beseg};
  for (void* p : ps) if (p) dfree(p);
  C = Cand{};
}
static void ensure_cands(gq_ctx* c, int n) {
  if (n <= c->C.cap) return;
  // candidates of a stage are rebuilt from scratch, so growth may drop contents
  free_cands(c->C);
  alloc_cands(c, std::max(n, 2 * c->C.cap), 256);
}
// grow keeping the first n_keep candidates (redirects are appended mid-round)
static void grow_cands_keep(gq_ctx* c, int need, int n_keep) {
  if (need <= c->C.cap) return;
  Cand old = c->C;
  c->C = Cand{};
  alloc_cands(c, std::max(need, 2 * old.cap), old.nbigcap);
  Cand& C = c->C;
  size_t k = (size_t)n_keep;
#define CPY(f, w) CK(cudaMemcpy(C.f, old.f, sizeof(*old.f) * (w) * k, cudaMemcpyDeviceToDevice))
  CPY(kind, 1); CPY(tgt, 1); CPY(seed, 1); CPY(status, 1); CPY(memb, 1); CPY(pool, 1); CPY(rank, 1);
  CPY(allow, 1); CPY(nallow, 1); CPY(extra, 1); CPY(p, 3); CPY(h, 1); CPY(canon, 1); CPY(state, 1);
  CPY(vid, 1); CPY(nt0, 1); CPY(ntet, 1); CPY(nbf, 1); CPY(ncr, 1); CPY(nbsub, 1); CPY(nbseg, 1);
  CPY(neseg, 1); CPY(mind, 1); CPY(tets, CT); CPY(bf, CF); CPY(cr, CC); CPY(crf, CC); CPY(bsub, CC);
  CPY(bseg, CC); CPY(eseg, CC); CPY(rseg, CRD); CPY(rface, CRD); CPY(nrseg, 1); CPY(nrface, 1); CPY(bigi, 1);
#undef CPY
  size_t kb = (size_t)old.nbigcap;
  CK(cudaMemcpy(C.btets, old.btets, 4 * kb * CTB, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(C.bbf, old.bbf, 4 * kb * CFB, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(C.bcr, old.bcr, 4 * kb * CCB, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(C.bcrf, old.bcrf, 4 * kb * CCB, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(C.bbsub, old.bbsub, 4 * kb * CCB, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(C.bbseg, old.bbseg, 4 * kb * CCB, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(C.beseg, old.beseg, 4 * kb * CCB, cudaMemcpyDeviceToDevice));
  free_cands(old);
}
// big-region slabs: grow keeping the first c->big_used ones
static void ensure_big(gq_ctx* c, int need) {
  Cand& C = c->C;
  if (need <= C.nbigcap) return;
  int cap = std::max(need, 2 * C.nbigcap);
  size_t keep = (size_t)c->big_used;
  auto grow = [&](int*& ptr, size_t w) {
    int* q = dmalloc<int>((size_t)cap * w);
    if (keep) CK(cudaMemcpy(q, ptr, 4 * keep * w, cudaMemcpyDeviceToDevice));
    dfree(ptr);
    ptr = q;
  };
  grow(C.btets, CTB); grow(C.bbf, CFB); grow(C.bcr, CCB); grow(C.bcrf, CCB);
  grow(C.bbsub, CCB); grow(C.bbseg, CCB); grow(C.beseg, CCB);
  C.nbigcap = cap;
}
// 2D retiling work items (candidate, polygon): grown on demand (facet-heavy rounds)
static void ensure_items(gq_ctx* c, int n) {
  if (n <= c->T.icap) return;
  int icap = std::max(n, 2 * c->T.icap);
  for (int** q : {&c->T.cand, &c->T.pid, &c->T.state, &c->T.ncav, &c->T.nrem}) { dfree(*q); *q = dmalloc<int>(icap); }
  dfree(c->T.cav); c->T.cav = dmalloc<int>((size_t)icap * c->T.cap);
  dfree(c->T.rem); c->T.rem = dmalloc<int>((size_t)icap * c->T.rcap);
  c->T.icap = icap;
}
static unsigned int pow2_at_least(size_t n) { unsigned int p = 1024; while (p < n) p <<= 1; return p; }

static void alloc_mesh(gq_ctx* c, int n, int m, int f, int npidx) {
  Dev& D = c->D;
  size_t vcap = 65536 + (size_t)n * 8;
  size_t tcap = std::max<size_t>(1 << 21, (size_t)n * 64);
  D.vcap = (int)vcap; D.tcap = (int)tcap;
  D.P = dmalloc<double>(3 * vcap); D.vorigin = dmalloc<uint8_t>(vcap); D.vert_tet = dmalloc<int>(vcap);
  D.vsid = dmalloc<int>(vcap);
  D.tv = dmalloc<int4>(tcap); D.tn = dmalloc<int4>(tcap); D.alive = dmalloc<uint8_t>(tcap);
  D.sub = dmalloc<uint8_t>(tcap); D.seg = dmalloc<uint8_t>(tcap); D.skip = dmalloc<uint8_t>(tcap);
  D.ratio = dmalloc<double>(tcap);
  CK(cudaMemset(D.alive, 0, tcap));
  if (getenv("GQ_PROFILE")) std::fprintf(stderr, "[gq] capacities: verts %zu tets %zu\n", vcap, tcap);
  size_t sgcap = 65536 + (size_t)m * 32 + vcap / 8;
  D.sgcap = (int)sgcap;
  D.sg_uv = dmalloc<int2>(sgcap); D.sg_sid = dmalloc<int>(sgcap); D.sg_fl = dmalloc<unsigned int>(sgcap);
  unsigned int sgh = pow2_at_least(2 * sgcap);
  D.sg_hk = dmalloc<unsigned long long>(sgh); D.sg_hv = dmalloc<int>(sgh); D.sg_hmask = sgh - 1;
  CK(cudaMemset(D.sg_hk, 0xff, (size_t)sgh * 8));
  size_t sfcap = 65536 + (size_t)npidx * 32 + vcap;
  D.sfcap = (int)sfcap;
  D.sf_v = dmalloc<int4>(sfcap); D.sf_fl = dmalloc<unsigned int>(sfcap);
  unsigned int sfh = pow2_at_least(2 * sfcap);
  D.sf_hk = dmalloc<unsigned long long>(sfh); D.sf_hv = dmalloc<int>(sfh); D.sf_hmask = sfh - 1;
  CK(cudaMemset(D.sf_hk, 0xff, (size_t)sfh * 8));
  size_t t2cap = 65536 + (size_t)npidx * 8 + 2 * vcap;
  D.t2cap = (int)t2cap;
  D.t2v = dmalloc<int4>(t2cap); D.t2alive = dmalloc<uint8_t>(t2cap);
  CK(cudaMemset(D.t2alive, 0, t2cap));
  unsigned int heh = pow2_at_least(4 * t2cap);
  D.he_hk = dmalloc<unsigned long long>(heh); D.he_hv = dmalloc<int>(heh); D.he_hmask = heh - 1;
  CK(cudaMemset(D.he_hk, 0xff, (size_t)heh * 8));
  D.t2count = dmalloc<int>(std::max(f, 1));
  CK(cudaMemset(D.t2count, 0, std::max(f, 1) * 4));
  D.poly_keep = dmalloc<int2>(std::max(f, 1));
  D.poly_obl = dmalloc<uint8_t>(std::max(f, 1));
  D.t2last = dmalloc<int>(std::max(f, 1));
  CK(cudaMemset(D.t2last, 0xff, 4 * (size_t)std::max(f, 1)));
  D.segpoly_off = dmalloc<int>(m + 1);
  D.segpoly = dmalloc<int>(std::max(npidx, 1));
  D.sid_uv = dmalloc<int2>(std::max(m, 1));
  D.nsid = m; D.npoly = f;
  c->dctr = dmalloc<Counters>(1);
  D.ctr = c->dctr;
  // filter owners: [tets | faces | seg records]
  c->W.toff = 0; c->W.foff = (int)tcap; c->W.soff = (int)(5 * tcap);
  c->W.own = dmalloc<int>(5 * tcap + sgcap);
  CK(cudaMemset(c->W.own, 0x7f, (5 * tcap + sgcap) * 4));
  // 2D items
  c->T.cap = 256; c->T.rcap = 128;
  c->T.icap = 0;
  c->T.cand = c->T.pid = c->T.state = c->T.ncav = c->T.nrem = c->T.cav = c->T.rem = nullptr;   // freed by free_all
  ensure_items(c, 1 << 16);
  c->T.own = dmalloc<int>(t2cap);
  CK(cudaMemset(c->T.own, 0x7f, t2cap * 4));
  c->L.cap = 1 << 20; c->L.rows = dmalloc<int>((size_t)8 * c->L.cap);
  c->d_int = dmalloc<int>(64);
  alloc_scratch(c->S, 16384, CT * 2, 1024, 2048);
  alloc_scratch(c->SB, 512, CTB * 2, 32768, 32768);
  alloc_cands(c, 1 << 16, 256);
  {
    int g = (int)std::cbrt(std::max(1.0, n / 2.0));
    g = std::min(std::max(g, 4), 160);
    c->G.G = g;
    size_t ncell = 0;
    c->G.L = 0;
    for (int l = 0;; ++l) {
      int gl = cg_gl(g, l);
      c->G.off[l] = (int)ncell;
      ncell += (size_t)gl * gl * gl;
      c->G.L = l + 1;
      if (gl == 1) break;
    }
    c->G.ncell = (int)ncell;
    c->G.start = dmalloc<int>(ncell + 1);
    c->G.cnt = dmalloc<int>(ncell + 1);
    c->G.node_cap = (int)std::min<size_t>(((size_t)sgcap + sfcap) * 27, (size_t)1 << 30);
    c->G.codes = dmalloc<int>(c->G.node_cap);
    c->G.nbig = dmalloc<int>(2);
    c->reg_seg = c->reg_face = 0;
  }
  c->allocated = true;
}

static void free_all(gq_ctx* c) {
  if (!c->allocated) return;
  Dev& D = c->D;
  void* ps[] = {D.P, D.vorigin, D.vert_tet, D.vsid, D.tv, D.tn, D.alive, D.sub, D.seg, D.skip, D.ratio, D.sg_uv,
                D.sg_sid, D.sg_fl, D.sg_hk, D.sg_hv, D.sf_v, D.sf_fl, D.sf_hk, D.sf_hv, D.t2v, D.t2alive, D.he_hk,
                D.he_hv, D.t2count, D.poly_keep, D.poly_obl, D.t2last, D.segpoly_off, D.segpoly, D.sid_uv, c->dctr, c->W.own, c->T.cand,
                c->T.pid, c->T.state, c->T.cav, c->T.ncav, c->T.rem, c->T.nrem, c->T.own, c->L.rows, c->d_int,
                c->S.tkey, c->S.tval, c->S.tep, c->S.fkey, c->S.fep, c->S.epoch, c->S.list, c->S.stack, c->S.in,
                c->S.comp, c->SB.tkey, c->SB.tval, c->SB.tep, c->SB.fkey, c->SB.fep, c->SB.epoch, c->SB.list,
                c->SB.stack, c->SB.in, c->SB.comp, c->tmpA, c->tmpB, c->tmpC, c->k64a, c->k64b, c->k32a, c->k32b,
                c->cub_tmp, c->d_order, c->G.start, c->G.codes, c->G.cnt, c->G.nbig, c->Q.a, c->Q.b, c->Q.c,
                c->Q.d, c->Q.e, c->Q.f, c->Q.g, c->Q.h, c->tv2, c->tn2, c->sub2, c->seg2, c->skip2, c->ratio2};
  for (void* p : ps) if (p) dfree(p);
  free_cands(c->C);
  c->allocated = false;
  c->tmpcap = 0; c->cub_cap = 0; c->cub_tmp = nullptr;
  c->tmpA = c->tmpB = c->tmpC = nullptr; c->k64a = c->k64b = nullptr; c->k32a = c->k32b = nullptr; c->d_order = nullptr;
  c->Q = {};
  c->tv2 = c->tn2 = nullptr; c->sub2 = c->seg2 = c->skip2 = nullptr; c->ratio2 = nullptr;
}

// regions for candidates [n0,n1): normal pass, then the overflow ones with big slabs
static cudaEvent_t ev_next(gq_ctx* c) {
  if (c->evused == c->evpool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->evpool.push_back(e);
  }
  return c->evpool[c->evused++];
}
static void region_begin(gq_ctx* c) { c->er0 = ev_next(c); CK(cudaEventRecord(c->er0, c->st)); }
static void region_end(gq_ctx* c) {
  c->er1 = ev_next(c);
  CK(cudaEventRecord(c->er1, c->st));
  c->rpairs.push_back({c->er0, c->er1});
}
// after the final sync of a refine: sum the region-kernel intervals, resolve the stage timeline
static void resolve_events(gq_ctx* c) {
  for (auto& pr : c->rpairs) { float ms = 0; cudaEventElapsedTime(&ms, pr.first, pr.second); c->region_ms += ms; }
  for (size_t i = 1; i < c->fev.size(); ++i) {
    if (c->fev[i].second < 0) continue;
    float ms = 0;
    cudaEventElapsedTime(&ms, c->fev[i - 1].first, c->fev[i].first);
    g_fine_t[c->fev[i].second] += ms * 1e-3;
  }
  c->rpairs.clear(); c->fev.clear(); c->evused = 0;
}
template <class K>
static void launch_warp_regions(gq_ctx* c, K kern, size_t shm, int nwork, int n0, int n1, const int* list) {
  int blocks = (int)std::min<long long>(((long long)nwork + WR_WARPS - 1) / WR_WARPS, c->S.nthreads / WR_WARPS);
  kern<<<std::max(blocks, 1), 32 * WR_WARPS, shm, c->st>>>(c->D, c->C, c->S, n0, n1, list);
  c->launches++;
  CK(cudaGetLastError());
}
static void run_regions(gq_ctx* c, int n0, int n1, int probe) {
  if (n1 <= n0) return;
  fine(c, 31);
  region_begin(c);
  if (!getenv("GQ_THREAD_REGIONS")) {   // debug switch: per-thread kernel
    launch_warp_regions(c, k_region_warp<WT1_MAXT, WT1_HASH, WT1_MINB>, WR_WARPS * sizeof(WarpShared1), n1 - n0, n0, n1,
                        (const int*)nullptr);
  } else {
    LAUNCH_S(k_region, n1 - n0, c->D, c->C, c->S, n0, n1, (const int*)nullptr, probe, 0);
  }
  region_end(c);
  if (g_trace) {   // per-launch algorithmic bytes for matching an ncu capture
    static long long launch_no = 0;
    static unsigned long long t_last = 0, r_last = 0;
    sync(c);
    unsigned long long rc = 0, tested = 0;
    CK(cudaMemcpyFromSymbol(&rc, g_region_calls, 8));
    CK(cudaMemcpyFromSymbol(&tested, g_tested, 8));
    float ms = 0; cudaEventElapsedTime(&ms, c->er0, c->er1);
    std::fprintf(stderr, "[region] launch %lld cands %d bytes_alg %llu ms %.3f\n", launch_no++, n1 - n0,
                 58ull * (tested - t_last) + 24ull * (rc - r_last), ms);
    t_last = tested; r_last = rc;
  }
  fine(c, 24);
  // overflow passes: the large warp tier, then one block per cavity
  ensure_tmp(c, n1 + 1);
  std::vector<int> hs(n1 - n0);
  CK(cudaMemcpyAsync(hs.data(), c->C.status + n0, sizeof(int) * (n1 - n0), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  std::vector<int> ovf;
  for (int k = 0; k < n1 - n0; ++k) if (hs[k] == CS_OVF) ovf.push_back(n0 + k);
  std::vector<int> big;
  if (!ovf.empty() && WT1_MAXT != WT2_MAXT && !getenv("GQ_THREAD_REGIONS")) {
    int no = (int)ovf.size();
    CK(cudaMemcpyAsync(c->tmpB, ovf.data(), sizeof(int) * no, cudaMemcpyHostToDevice, c->st));
    region_begin(c);
    launch_warp_regions(c, k_region_warp<WT2_MAXT, WT2_HASH, 1>, WR_WARPS * sizeof(WarpShared2), no, 0, no, c->tmpB);
    region_end(c);
    LAUNCH(k_gather_status, no, c->C, c->tmpB, no, c->tmpA);
    CK(cudaMemcpyAsync(hs.data(), c->tmpA, sizeof(int) * no, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int k = 0; k < no; ++k) if (hs[k] == CS_OVF) big.push_back(ovf[k]);
  } else {
    big.swap(ovf);
  }
  fine(c, 25);
  if (!big.empty()) {
    int nb = (int)big.size();
    ensure_big(c, c->big_used + nb);
    CK(cudaMemcpyAsync(c->tmpC, big.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, c->st));
    k_region_block<<<std::min(nb, c->SB.nthreads), BR_THREADS, sizeof(BlockShared), c->st>>>(c->D, c->C, c->SB, c->tmpC, nb, c->big_used);
    c->launches++;
    CK(cudaGetLastError());
    c->big_used += nb;
    double tb = now_s();
    sync(c);
    if (g_trace) {
      std::vector<int> nts(nb);
      int mx = 0; long long sm = 0;
      for (int k = 0; k < nb; ++k) {
        CK(cudaMemcpy(&nts[k], c->C.ntet + big[k], 4, cudaMemcpyDeviceToHost));
        mx = std::max(mx, nts[k]); sm += nts[k];
      }
      std::fprintf(stderr, "[big] n %d of %d tets max %d mean %.0f block %.3f ms\n", nb, n1 - n0, mx, (double)sm / nb, 1e3 * (now_s() - tb));
    }
  }
  fine(c, 26);
}

// candidates sorted by priority (class rank, hash); smaller first
// (refine.py:45-52).  Equal hashes would fall back to the canonical tuple in
// the reference; a 64-bit splitmix collision inside one round is ignored.
__global__ void k_rank_keys(Cand C, int n, unsigned long long* kh, unsigned int* kk, int* idx) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    bool ok = C.status[c] == CS_OK;
    kh[c] = ok ? C.h[c] : ~0ull;
    kk[c] = ok ? (unsigned int)C.kind[c] : 7u;
    idx[c] = c;
  }
}
static void rank_candidates(gq_ctx* c, int n) {
  if (n <= 0) return;
  ensure_tmp(c, n + 1);
  LAUNCH(k_rank_keys, n, c->C, n, c->k64a, c->k32a, c->tmpA);
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, c->k64a, c->k64b, c->tmpA, c->tmpB, n, 0, 64, c->st);
  ensure_cub(c, need);
  cub::DeviceRadixSort::SortPairs(c->cub_tmp, need, c->k64a, c->k64b, c->tmpA, c->tmpB, n, 0, 64, c->st);
  LAUNCH(k_gather_u32, n, c->k32a, c->tmpB, n, c->k32b);
  need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, c->k32b, c->k32a, c->tmpB, c->tmpA, n, 0, 3, c->st);
  ensure_cub(c, need);
  cub::DeviceRadixSort::SortPairs(c->cub_tmp, need, c->k32b, c->k32a, c->tmpB, c->tmpA, n, 0, 3, c->st);
  LAUNCH(k_rank_scatter, n, c->C, c->tmpA, n);
}

// LFMIS filter over candidates [0,n): state 0 for ok ones, 3 for the rest.
static void run_filter(gq_ctx* c, int n, int* nacc_out) {
  if (n <= 0) return;
  if (!getenv("GQ_FILTER_LAUNCHES")) {
    static int blocks_per_sm = 0, nsm = 0;
    if (!blocks_per_sm) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_filter_coop, 256, 0));
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      if (blocks_per_sm < 1) throw std::runtime_error("filter kernel cannot be resident");
    }
    int blocks = std::min(blocks_per_sm * nsm, (n + 7) / 8);
    int* ctr = c->d_int + 48;
    CK(cudaMemsetAsync(ctr, 0, 12, c->st));
    void* args[] = {&c->D, &c->C, &c->W, &n, &ctr};
    CK(cudaLaunchCooperativeKernel((void*)k_filter_coop, dim3(std::max(blocks, 1)), dim3(256), args, 0, c->st));
    c->launches++;
    return;
  }
  // debug path: one launch per pass, iterations are idempotent once nothing is undecided: check every 3rd
  for (int it = 0;; ++it) {
    CK(cudaMemsetAsync(c->d_int, 0, 4, c->st));
    LAUNCH(k_claim, n, c->D, c->C, c->W, n);
    LAUNCH(k_decide, n, c->D, c->C, c->W, n, it);
    LAUNCH(k_mark, n, c->D, c->C, c->W, n, it);
    LAUNCH(k_reject, n, c->D, c->C, c->W, n, c->d_int);
    LAUNCH(k_reset_claims, n, c->D, c->C, c->W, n, 0);
    if (it % 3 != 2) continue;
    int und = read_int(c, c->d_int);
    if (und == 0) break;
    if (it > 100000) throw std::runtime_error("filter did not converge");
  }
  LAUNCH(k_reset_claims, n, c->D, c->C, c->W, n, 1);
  (void)nacc_out;
}

// bulk construction: a point goes in this round only if no lower-order
// pending point claims any of its elements (so it commutes with all of them)
static void run_filter_strict(gq_ctx* c, int n) {
  LAUNCH(k_claim, n, c->D, c->C, c->W, n);
  LAUNCH(k_decide, n, c->D, c->C, c->W, n, 0);
  LAUNCH(k_reset_claims, n, c->D, c->C, c->W, n, 1);
  LAUNCH(k_strict_state, n, c->C, n);
}

// live records of a phase with all `need` flags and none of `deny`, sorted
// by vertex key (refine.py:587, 595: sorted(enc_* - blocked_*)); ids -> out
static int sorted_records(gq_ctx* c, int phase, unsigned int need, unsigned int deny, int* out) {
  int n = phase == 0 ? c->hc.nsegrec : c->hc.nfacerec;
  if (n <= 0) return 0;
  ensure_tmp(c, n + 1);
  LAUNCH(k_flag_pending_keys, n, c->D, phase, need, deny, c->Q.e, c->k64a, c->k32a);
  int cnt = select_flagged(c, c->Q.e, n, c->tmpA);       // record ids, ascending
  if (cnt == 0) return 0;
  size_t nb = 0;
  if (phase == 0) {
    LAUNCH(k_gather_u64, cnt, c->k64a, c->tmpA, cnt, c->k64b);
    cub::DeviceRadixSort::SortPairs(nullptr, nb, c->k64b, c->k64a, c->tmpA, out, cnt, 0, 64, c->st);
    ensure_cub(c, nb);
    cub::DeviceRadixSort::SortPairs(c->cub_tmp, nb, c->k64b, c->k64a, c->tmpA, out, cnt, 0, 64, c->st);
  } else {
    // (b,c) then a: two stable passes
    LAUNCH(k_gather_u64, cnt, c->k64a, c->tmpA, cnt, c->k64b);
    cub::DeviceRadixSort::SortPairs(nullptr, nb, c->k64b, c->k64a, c->tmpA, c->tmpB, cnt, 0, 64, c->st);
    ensure_cub(c, nb);
    cub::DeviceRadixSort::SortPairs(c->cub_tmp, nb, c->k64b, c->k64a, c->tmpA, c->tmpB, cnt, 0, 64, c->st);
    LAUNCH(k_face_a, cnt, c->D, c->tmpB, cnt, c->k32b);
    nb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, nb, c->k32b, c->k32a, c->tmpB, out, cnt, 0, 32, c->st);
    ensure_cub(c, nb);
    cub::DeviceRadixSort::SortPairs(c->cub_tmp, nb, c->k32b, c->k32a, c->tmpB, out, cnt, 0, 32, c->st);
  }
  return cnt;
}

// register records created since the last call (ConstraintIndex.add_*)
static void grid_sync(gq_ctx* c) {
  pull(c);
  int nseg = c->hc.nsegrec, nface = c->hc.nfacerec, ncell = c->G.ncell;
  CK(cudaMemsetAsync(c->G.cnt, 0, 4 * (size_t)(ncell + 1), c->st));   // slot ncell stays 0: start[ncell] = total
  CK(cudaMemsetAsync(c->G.nbig, 0, 8, c->st));
  if (nseg + nface > 0) LAUNCH(k_grid_build, nseg + nface, c->D, c->G, nseg, nface, 0);
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, c->G.cnt, c->G.start, ncell + 1, c->st);
  ensure_cub(c, need);
  cub::DeviceScan::ExclusiveSum(c->cub_tmp, need, c->G.cnt, c->G.start, ncell + 1, c->st);
  CK(cudaMemsetAsync(c->G.cnt, 0, 4 * (size_t)ncell, c->st));
  if (nseg + nface > 0) LAUNCH(k_grid_build, nseg + nface, c->D, c->G, nseg, nface, 1);
}

static bool full_verify(gq_ctx* c) {
  CK(cudaMemsetAsync(c->d_int, 0, 16, c->st));
  pull(c);
  LAUNCH_S(k_check, c->hc.nsegrec + c->hc.nfacerec, c->D, c->S, 1, c->d_int);
  LAUNCH(k_clear_flag, c->hc.nsegrec + c->hc.nfacerec, c->D, RF_BLOCK);
  CK(cudaMemsetAsync(c->d_int + 4, 0, 16, c->st));
  LAUNCH(k_count_pending, c->hc.nsegrec + c->hc.nfacerec, c->D, c->d_int + 4);
  int h[8];
  CK(cudaMemcpyAsync(h, c->d_int, 32, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return h[0] > 0 || h[6] > 0 || h[7] > 0;
}

static void compact_tets(gq_ctx* c) {
  pull(c);
  int nt = c->hc.nt;
  ensure_tmp(c, nt + 1);
  LAUNCH(k_compact_flags, nt, c->D, c->tmpA);
  exclusive_scan(c, c->tmpA, c->tmpB, nt);
  int last_flag = read_int(c, c->tmpA + nt - 1), last_scan = read_int(c, c->tmpB + nt - 1);
  int na = last_scan + last_flag;
  Dev& D = c->D;
  // double buffers, allocated once per context
  if (!c->tv2) {
    c->tv2 = dmalloc<int4>(D.tcap); c->tn2 = dmalloc<int4>(D.tcap);
    c->sub2 = dmalloc<uint8_t>(D.tcap); c->seg2 = dmalloc<uint8_t>(D.tcap);
    c->ratio2 = dmalloc<double>(D.tcap); c->skip2 = dmalloc<uint8_t>(D.tcap);
  }
  LAUNCH(k_compact_move, nt, D, c->tmpB, nt, c->tv2, c->tn2, c->sub2, c->seg2, c->ratio2, c->skip2);
  LAUNCH(k_compact_vt, c->hc.nv, D, c->tmpB, c->tmpA, c->hc.nv);
  std::swap(D.tv, c->tv2); std::swap(D.tn, c->tn2); std::swap(D.sub, c->sub2); std::swap(D.seg, c->seg2);
  std::swap(D.ratio, c->ratio2); std::swap(D.skip, c->skip2);
  CK(cudaMemsetAsync(D.alive, 0, nt, c->st));
  CK(cudaMemsetAsync(D.alive, 1, na, c->st));
  c->hc.nt = na;
  push(c);
}

static void ensure_big(gq_ctx* c, int need);
static void init_delaunay(gq_ctx* c, const int* order, int n) {
  CK(cudaMemcpyAsync(c->d_order, order, 4 * (size_t)n, cudaMemcpyHostToDevice, c->st));
  LAUNCH(k_init_first, 1, c->D, c->d_order, n, c->d_int + 8);
  sync(c);
  int first[4];
  CK(cudaMemcpy(first, c->d_int + 8, 16, cudaMemcpyDeviceToHost));
  std::vector<int> pend;
  pend.reserve(n);
  for (int k = 0; k < n; ++k) {
    int v = order[k];
    if (v == first[0] || v == first[1] || v == first[2] || v == first[3]) continue;
    pend.push_back(v);
  }
  int np = (int)pend.size();
  if (np == 0) return;
  ensure_cands(c, np);
  Cand& C = c->C;
  int* d_pend = dmalloc<int>(np);
  int* d_hint = dmalloc<int>(np);
  int* d_plist = dmalloc<int>(np);
  int* d_plist2 = dmalloc<int>(np);
  int* d_acc = dmalloc<int>(np);
  int* d_scan = dmalloc<int>(np);
  int* d_keep = dmalloc<int>(np);
  int* d_succ = dmalloc<int>(c->D.tcap);
  int* d_touched = dmalloc<int>(c->D.tcap);
  CK(cudaMemsetAsync(d_succ, 0xff, 4 * (size_t)c->D.tcap, c->st));
  CK(cudaMemsetAsync(d_touched, 0xff, 4 * (size_t)c->D.tcap, c->st));
  CK(cudaMemsetAsync(d_hint, 0xff, 4 * (size_t)np, c->st));   // -1: no walk yet
  CellHint H;
  {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    std::vector<double> P(3 * (size_t)n);
    CK(cudaMemcpy(P.data(), c->D.P, 24 * (size_t)n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], P[3 * i + k]); hi[k] = std::max(hi[k], P[3 * i + k]); }
    H.G = std::max(1, std::min(128, (int)std::cbrt(n / 2.0)));
    for (int k = 0; k < 3; ++k) { H.lo[k] = lo[k]; H.inv[k] = hi[k] > lo[k] ? H.G / (hi[k] - lo[k]) : 0.0; }
    H.cellv = dmalloc<int>((size_t)H.G * H.G * H.G);
    CK(cudaMemsetAsync(H.cellv, 0xff, 4 * (size_t)H.G * H.G * H.G, c->st));
  }
  CK(cudaMemsetAsync(C.status, 0, 4 * (size_t)np, c->st));          // CS_OK, not cached
  CK(cudaMemsetAsync(C.memb, 0xff, 4 * (size_t)np, c->st));
  CK(cudaMemsetAsync(C.bigi, 0xff, 4 * (size_t)np, c->st));
  CK(cudaMemcpyAsync(d_pend, pend.data(), 4 * (size_t)np, cudaMemcpyHostToDevice, c->st));
  std::vector<int> ident(np);
  for (int k = 0; k < np; ++k) ident[k] = k;
  CK(cudaMemcpyAsync(d_plist, ident.data(), 4 * (size_t)np, cudaMemcpyHostToDevice, c->st));
  pull(c);
  int nt = c->hc.nt;
  int left = np, inserted = 4;
  // window = the next wf * inserted pending points; the number of rounds is set by the
  // strict-order dependency chain, not the window, so a small window only saves work
  double wf = getenv("GQ_INIT_WINDOW") ? atof(getenv("GQ_INIT_WINDOW")) : 0.0625;
  fine(c, -1);
  for (int round = 0; left > 0; ++round) {
    int W = (int)std::min<double>(left, std::max(64.0, wf * inserted));
    fine(c, 22);
    region_begin(c);
    if (!getenv("GQ_THREAD_INIT")) {
      int blocks = std::min((W + WR_WARPS - 1) / WR_WARPS, c->S.nthreads / WR_WARPS);
      static int* h_wdbg = nullptr;
      if (getenv("GQ_WATCHDOG") && !h_wdbg) {
        CK(cudaHostAlloc(&h_wdbg, 200000 * sizeof(int), cudaHostAllocMapped));
        int* dptr; CK(cudaHostGetDevicePointer(&dptr, h_wdbg, 0));
        CK(cudaMemcpyToSymbol(g_wdbg, &dptr, sizeof(dptr)));
      }
      if (h_wdbg) std::memset(h_wdbg, 0xff, 200000 * sizeof(int));
      k_init_region_warp<WT1_MAXT, WT1_HASH, WT1_MINB><<<std::max(blocks, 1), 32 * WR_WARPS, WR_WARPS * sizeof(WarpShared1), c->st>>>(
          c->D, C, c->S, d_pend, d_plist, W, d_hint, d_succ, d_touched, round, H, 0);
      c->launches++;
      CK(cudaGetLastError());
      if (h_wdbg) {
        CK(cudaEventRecord(c->er1, c->st));
        double t0w = now_s();
        while (cudaEventQuery(c->er1) == cudaErrorNotReady && now_s() - t0w < 5.0) {}
        if (cudaEventQuery(c->er1) == cudaErrorNotReady) {
          int shown = 0, nstart = 0, ndone = 0;
          for (int g = 0; g < 2 * 16384; g += 2) { nstart += h_wdbg[g] >= 0; ndone += h_wdbg[g + 1] == 99; }
          std::fprintf(stderr, "[watchdog] round %d W %d warps started %d at-99 %d\n", round, W, nstart, ndone);
          for (int g = 0; g < 2 * 16384 && shown < 20; g += 2) {
            if (h_wdbg[g] >= 0 && h_wdbg[g + 1] != 99) { std::fprintf(stderr, "[watchdog] round %d warp %d cand %d stage %d\n", round, g / 2, h_wdbg[g], h_wdbg[g + 1]); ++shown; }
          }
          for (int g = 0; g < 64 * 32; ++g) if (h_wdbg[40000 + g] >= 0) std::fprintf(stderr, "%d:%d ", g, h_wdbg[40000 + g]);
          std::fprintf(stderr, "\n[watchdog] kernel stuck; exiting\n");
          std::_Exit(3);
        }
      }
    } else {
      LAUNCH_S(k_init_region, W, c->D, C, c->S, d_pend, d_plist, W, d_hint, d_succ, d_touched, round, 0);
    }
    region_end(c);
    fine(c, 0);
    // big cavities (early rounds): resolve the lowest-order ones, truncate the window at the rest
    std::vector<int> bl;
    {
      CK(cudaMemsetAsync(c->d_int + 40, 0, 8, c->st));
      LAUNCH(k_count_ovf, W, C, d_plist, W, c->d_int + 40);
      int novf = read_int(c, c->d_int + 40);
      if (novf > 0) {
        std::vector<int> pl(W), sw(W);
        LAUNCH(k_gather_status, W, C, d_plist, W, d_scan);
        CK(cudaMemcpyAsync(pl.data(), d_plist, 4 * (size_t)W, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(sw.data(), d_scan, 4 * (size_t)W, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        for (int w = 0; w < W; ++w) if (sw[w] == CS_OVF) bl.push_back(pl[w]);
        if (WT1_MAXT != WT2_MAXT && !getenv("GQ_THREAD_INIT")) {   // the large warp tier first
          int no = (int)bl.size();
          CK(cudaMemcpyAsync(d_keep, bl.data(), 4 * (size_t)no, cudaMemcpyHostToDevice, c->st));
          int blocks = std::min((no + WR_WARPS - 1) / WR_WARPS, c->S.nthreads / WR_WARPS);
          k_init_region_warp<WT2_MAXT, WT2_HASH, 1><<<std::max(blocks, 1), 32 * WR_WARPS, WR_WARPS * sizeof(WarpShared2), c->st>>>(
              c->D, C, c->S, d_pend, d_keep, no, d_hint, d_succ, d_touched, round, H, 1);
          c->launches++;
          CK(cudaGetLastError());
          LAUNCH(k_gather_status, no, C, d_keep, no, d_scan);
          std::vector<int> s2(no);
          CK(cudaMemcpyAsync(s2.data(), d_scan, 4 * (size_t)no, cudaMemcpyDeviceToHost, c->st));
          sync(c);
          std::vector<int> rest;
          for (int k = 0; k < no; ++k) if (s2[k] == CS_OVF) rest.push_back(bl[k]);
          bl.swap(rest);
        }
        int nb = (int)std::min<size_t>(bl.size(), 4096);
        bl.resize(nb);
        if (nb > 0) {
        ensure_big(c, nb);
        ensure_tmp(c, nb + 1);
        std::vector<int> bis(nb);
        for (int k = 0; k < nb; ++k) bis[k] = k;
        CK(cudaMemcpyAsync(d_keep, bl.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(d_acc, bis.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, c->st));
        LAUNCH(k_scatter_ints, nb, C.bigi, d_keep, d_acc, nb);
        CK(cudaMemcpyAsync(c->tmpA, bl.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, c->st));
        k_init_region_block<<<std::min(nb, c->SB.nthreads), BR_THREADS, sizeof(BlockShared), c->st>>>(c->D, C, c->SB, d_pend, c->tmpA, nb, d_hint, d_succ, round);
        c->launches++;
        CK(cudaGetLastError());
        LAUNCH(k_gather_status, W, C, d_plist, W, d_scan);
        CK(cudaMemcpyAsync(sw.data(), d_scan, 4 * (size_t)W, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        for (int w = 0; w < W; ++w) if (sw[w] == CS_OVF) { W = w; break; }
        if (W == 0) throw std::runtime_error("init: cavity overflow");
        CK(cudaMemcpyAsync(c->tmpC, bl.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, c->st));
        }
      }
    }
    fine(c, 1);
    int nacc = 0, add_t = 0;
    if (!getenv("GQ_INIT_LAUNCHES")) {
      static int bps = 0, nsm = 0;
      if (!bps) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_init_filter_coop, 256, 0));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        if (bps < 1) throw std::runtime_error("init filter kernel cannot be resident");
      }
      int blocks = std::max(1, std::min(bps * nsm, (W + 7) / 8));
      int* tot = c->d_int + 52;
      void* args[] = {&c->D, &C, &c->W, &d_plist, &W, &nt, &d_acc, &d_plist2, &d_scan, &tot, &d_succ};
      CK(cudaLaunchCooperativeKernel((void*)k_init_filter_coop, dim3(blocks), dim3(256), args, 0, c->st));
      c->launches++;
      int h2[2];
      CK(cudaMemcpyAsync(h2, tot, 8, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      nacc = h2[0]; add_t = h2[1];
      if (nt + add_t > c->D.tcap) throw std::runtime_error("tet capacity exceeded in init");
      fine(c, 3);
    } else {   // debug path: one launch per pass
      LAUNCH(k_init_claim, W, c->D, C, c->W, d_plist, W);
      LAUNCH(k_init_decide, W, c->D, C, c->W, d_plist, W, d_acc);
      LAUNCH(k_init_unclaim, W, c->D, C, c->W, d_plist, W);
      fine(c, 2);
      LAUNCH(k_init_nbf, W, C, d_plist, d_acc, W, d_keep);
      exclusive_scan(c, d_keep, d_scan, W);
      int lastn = 0, lasts = 0, lasta = 0;
      CK(cudaMemcpyAsync(&lastn, d_keep + W - 1, 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(&lasts, d_scan + W - 1, 4, cudaMemcpyDeviceToHost, c->st));
      exclusive_scan(c, d_acc, d_plist2, W);
      int lastacc_scan = 0;
      CK(cudaMemcpyAsync(&lastacc_scan, d_plist2 + W - 1, 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(&lasta, d_acc + W - 1, 4, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      nacc = lastacc_scan + lasta;
      add_t = lasts + lastn;
      if (nt + add_t > c->D.tcap) throw std::runtime_error("tet capacity exceeded in init");
      fine(c, 3);
      LAUNCH(k_init_kill, W, c->D, C, d_plist, d_acc, d_scan, W, nt, d_succ);
    }
    fine(c, 4);
    {
      int blocks = std::max(1, std::min((W + WS_WARPS - 1) / WS_WARPS, c->SB.nthreads / WS_WARPS));
      k_init_stars_warp<<<blocks, 32 * WS_WARPS, WS_WARPS * sizeof(StarShared), c->st>>>(c->D, C, d_pend, d_plist, d_acc, W, d_touched, round, c->SB);
      c->launches++;
      CK(cudaGetLastError());
    }
    fine(c, 5);
    LAUNCH(k_init_cellmark, W, c->D, H, d_pend, d_plist, d_acc, W);
    nt += add_t;
    // release big slabs (big regions are recomputed next round if still pending)
    {
      int* d_out = d_keep;   // the acceptance scan lives in d_plist2 (accscan)
      LAUNCH(k_init_compact2, left, d_plist, d_acc, d_plist2, W, left, nacc, d_out);
      std::swap(d_plist, d_keep);
    }
    if (!bl.empty()) LAUNCH(k_release_big, bl.size(), C, c->tmpC, (int)bl.size());
    if (g_trace) {
      sync(c);
      float rms = 0; cudaEventElapsedTime(&rms, c->rpairs.back().first, c->rpairs.back().second);
      unsigned long long rc = 0; CK(cudaMemcpyFromSymbol(&rc, g_region_calls, 8));
      static unsigned long long rc_last = 0;
      std::fprintf(stderr, "[init] round %d W %d big %d acc %d nt %d region_ms %.3f computed %llu maxtet %d\n", round, W,
                   (int)bl.size(), nacc, nt, rms, rc - rc_last, read_int(c, c->d_int + 41));
      rc_last = rc;
    }
    left -= nacc;
    inserted += nacc;
    c->hc.nt = nt;
    push(c);
    if (nacc == 0) throw std::runtime_error("init made no progress");
    c->init_rounds = round + 1;
    fine(c, 6);
  }
  // big-slab candidates must not keep stale bigi for the refinement rounds
  sync(c);
  dfree(d_pend); dfree(d_hint); dfree(d_plist); dfree(d_plist2); dfree(d_acc);
  dfree(d_scan); dfree(d_keep); dfree(d_succ); dfree(d_touched); dfree(H.cellv);
}

// ------------------------------------------------------------------ round

__global__ void k_states(Cand C, int n, int* okf, int* failf) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    int st = C.status[c];
    int s = st == CS_OK ? 0 : (st == CS_DROP ? -1 : 3);
    C.state[c] = s;
    okf[c] = s == 0;
    failf[c] = s == 3;
  }
}
__global__ void k_kept(Cand C, int n, int* keep) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) keep[c] = C.status[c] != CS_DROP;
}
__global__ void k_acc_byrank(Cand C, int n, int* byrank) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (C.state[c] == 1) byrank[C.rank[c]] = c;
}
__global__ void k_nonneg(const int* a, int n, int* f) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) f[i] = a[i] >= 0;
}
__global__ void k_gather_i32(const int* src, const int* idx, int n, int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}
__global__ void k_item_count(Dev D, Cand C, const int* ins, int ni, int* cnt) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ni; k += gridDim.x * blockDim.x) {
    int c = ins[k], kind = C.kind[c];
    if (kind == K_SEG) { int sid = D.sg_sid[C.tgt[c]]; cnt[k] = D.segpoly_off[sid + 1] - D.segpoly_off[sid]; }
    else cnt[k] = kind == K_FACE ? 1 : 0;
  }
}
__global__ void k_item_fill(Dev D, Cand C, const int* ins, int ni, const int* off, const int* cnt, T2Items T, int* item_of) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ni; k += gridDim.x * blockDim.x) {
    int c = ins[k], kind = C.kind[c], o = off[k];
    item_of[2 * k] = o; item_of[2 * k + 1] = o + cnt[k];
    if (kind == K_SEG) {
      int sid = D.sg_sid[C.tgt[c]];
      for (int j = 0; j < cnt[k]; ++j) { T.cand[o + j] = c; T.pid[o + j] = D.segpoly[D.segpoly_off[sid] + j]; T.state[o + j] = 0; T.nrem[o + j] = 0; }
    } else if (kind == K_FACE) {
      T.cand[o] = c; T.pid[o] = D.sf_v[C.tgt[c]].w; T.state[o] = 0; T.nrem[o] = 0;
    }
  }
}
__global__ void k_count_seed_dead(Dev D, Cand C, int n, int* out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 2 || C.kind[c] != K_TET) continue;
    atomicAdd(out, 1);
    if (!D.alive[C.tgt[c]]) atomicAdd(out + 1, 1);
  }
}
__global__ void k_bump(Dev D, int dnv, int dnt) { D.ctr->nv += dnv; D.ctr->nt += dnt; }
__global__ void k_pool_pos(Cand C, int n, const int* keepscan, const int* keep) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    C.pool[c] = keep[c] ? keepscan[c] : -1;
}

struct RoundOut { int phase = -1; long long ncand = 0, acc = 0, rej = 0, failed = 0, inserted = 0; };


static const char* g_prof_names[8] = {"pool", "regions", "filter", "insert", "2d", "fallback", "post", "other"};

// scan of n ints; returns the total
static int scan_total(gq_ctx* c, const int* in, int* out, int n) {
  if (n <= 0) return 0;
  exclusive_scan(c, in, out, n);
  int a = 0, b = 0;
  CK(cudaMemcpyAsync(&a, in + n - 1, 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(&b, out + n - 1, 4, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return a + b;
}

static void insert_accepted(gq_ctx* c, int n, long long* nacc_out, long long* inserted, int round_no) {
  Cand& C = c->C;
  double t0 = now_s();
  int* byrank = c->Q.a; int* flags = c->Q.b; int* pos = c->Q.c; int* acc = c->Q.d; int* ins = c->Q.e;
  CK(cudaMemsetAsync(byrank, 0xff, 4 * (size_t)n, c->st));
  LAUNCH(k_acc_byrank, n, C, n, byrank);
  LAUNCH(k_nonneg, n, byrank, n, flags);
  int na = select_flagged(c, flags, n, pos);
  *nacc_out = na;
  if (na == 0) return;
  LAUNCH(k_gather_i32, na, byrank, pos, na, acc);
  LAUNCH(k_accept_flags, na, c->D, C, acc, na, flags, c->L, round_no, c->D.lmin2);
  int ni = select_flagged(c, flags, na, pos);
  *inserted += ni;
  if (ni == 0) return;
  LAUNCH(k_gather_i32, ni, acc, pos, ni, ins);
  pull(c);
  int nv = c->hc.nv, nt = c->hc.nt;
  LAUNCH(k_gather_nbf, ni, C, ins, ni, flags);
  int tot = scan_total(c, flags, pos, ni);
  if (nt + tot > c->D.tcap || nv + ni > c->D.vcap) throw std::runtime_error("mesh capacity exceeded");
  LAUNCH(k_assign_ids, ni, C, ins, ni, pos, nv, nt);
  Ins I; I.list = ins; I.n = ni; I.nv0 = nv; I.nt0base = nt;
  fine(c, 18);
  LAUNCH(k_ins_vertices, ni, c->D, C, I);
  // facet 2D retiling work items (candidate, polygon) in priority order
  int* item_of = nullptr;
  int nit = 0;
  if (c->npoly > 0) {
    LAUNCH(k_item_count, ni, c->D, C, ins, ni, flags);
    nit = scan_total(c, flags, pos, ni);
    ensure_items(c, nit);
    item_of = c->Q.f;
    if (nit > 0) LAUNCH(k_item_fill, ni, c->D, C, ins, ni, pos, flags, c->T, item_of);
  }
  g_prof[3] += now_s() - t0;
  double t1 = now_s();
  if (nit > 0 && nit <= 512 && !getenv("GQ_T2_LAUNCHES")) {   // few items: all passes in one block
    c->T.n = nit;
    k_t2_fused<<<1, 128, 0, c->st>>>(c->D, C, c->T, c->S, c->d_int + 16);
    c->launches++;
    CK(cudaGetLastError());
  } else if (nit > 0) {
    c->T.n = nit;
    int left = nit;
    for (int pass = 0; left > 0; ++pass) {
      LAUNCH_S(k_t2_compute, nit, c->D, C, c->T, c->S);
      LAUNCH(k_t2_claim, nit, c->D, C, c->T);
      CK(cudaMemsetAsync(c->d_int + 16, 0, 4, c->st));
      LAUNCH_S(k_t2_apply, nit, c->D, C, c->T, c->S, c->d_int + 16);
      LAUNCH(k_t2_reset, nit, c->D, C, c->T, 1);
      LAUNCH_S(k_t2_commit, nit, c->D, C, c->T, c->S);
      LAUNCH(k_t2_retire, nit, c->D, c->T);
      int applied = read_int(c, c->d_int + 16);
      if (g_trace) std::fprintf(stderr, "[t2] pass %d applied %d of %d\n", pass, applied, left);
      left -= applied;
      if (applied == 0) throw std::runtime_error("2D retiling made no progress");
    }
  }
  g_prof[4] += now_s() - t1;
  if (g_trace && nit > 0) std::fprintf(stderr, "[t2] round %d items %d inserted %d\n", round_no, nit, ni);
  t1 = now_s();
  fine(c, 19);
  LAUNCH(k_ins_segsplit, ni, c->D, C, I);
  LAUNCH(k_kill_cavities, ni, c->D, C, I);
  {
    int blocks = std::max(1, std::min((ni + WS_WARPS - 1) / WS_WARPS, c->SB.nthreads / WS_WARPS));
    k_star_warp<<<blocks, 32 * WS_WARPS, WS_WARPS * sizeof(StarShared), c->st>>>(c->D, C, I, c->SB);
    c->launches++;
    CK(cudaGetLastError());
  }
  LAUNCH(k_bump, 1, c->D, ni, tot);
  fine(c, 20);
  LAUNCH_S(k_post_insert, ni, c->D, C, I, c->T, c->S, (const int*)item_of);
  fine(c, 21);
  g_prof[3] += now_s() - t1;
}

// appends the records flagged RF_REDIR of a phase as candidates (sorted)
static int append_redirects(gq_ctx* c, int phase, int at, int pool0, CandCtx X) {
  pull(c);
  int nr = sorted_records(c, phase, RF_REDIR, 0, c->Q.g);
  int nrec = phase == 0 ? c->hc.nsegrec : c->hc.nfacerec;
  if (nrec > 0) LAUNCH(k_clear_redir, nrec, c->D, phase);
  if (nr == 0) return 0;
  grow_cands_keep(c, at + nr, at);
  LAUNCH(k_set_cands, nr, c->C, at, nr, phase == 0 ? K_SEG : K_FACE, c->Q.g, pool0);
  LAUNCH_S(k_make_cands, nr, c->D, c->C, c->S, at, at + nr, X, c->L, c->D.lmin2);
  return nr;
}

static void ensure_q(gq_ctx* c, size_t n) {
  if (n <= c->Q.cap) return;
  int** ps[] = {&c->Q.a, &c->Q.b, &c->Q.c, &c->Q.d, &c->Q.e, &c->Q.f, &c->Q.g, &c->Q.h};
  size_t cap = n + n / 2;
  for (int** q : ps) { if (*q) dfree(*q); *q = dmalloc<int>(cap); }
  c->Q.cap = cap;
}

static void fine(gq_ctx* c, int k) {
  if (g_trace) { CK(cudaStreamSynchronize(c->st)); std::fprintf(stderr, "[trace] stage %d ok\n", k); }
  if (g_fine_ev) {
    cudaEvent_t e = ev_next(c);
    CK(cudaEventRecord(e, c->st));
    c->fev.push_back({e, k});
    return;
  }
  if (!g_fine) return;
  CK(cudaStreamSynchronize(c->st));
  double t = now_s();
  if (k >= 0) g_fine_t[k] += t - g_fine_last;
  g_fine_last = t;
}

static RoundOut run_round(gq_ctx* c, int round_no) {
  RoundOut R;
  c->big_used = 0;
  pull(c);
  ensure_q(c, (size_t)std::max(std::max(c->hc.nt, c->hc.nsegrec + c->hc.nfacerec), c->C.cap) * 2 + 4096);
  ensure_tmp(c, (size_t)std::max(std::max(c->hc.nt, c->hc.nsegrec + c->hc.nfacerec), c->C.cap) + 4096);
  double t0 = now_s();
  fine(c, -1);
  CandCtx X; X.round_no = round_no; X.seed = c->seed; X.with_facets = c->npoly > 0;
  double lmin2 = c->D.lmin2;
  int phase = -1, nbase = 0;
  int ns = sorted_records(c, 0, RF_ENC, RF_BLOCK | RF_SKIP, c->Q.g);
  fine(c, 11);
  if (ns > 0) {
    phase = 0;
    ensure_cands(c, ns);
    LAUNCH(k_set_cands, ns, c->C, 0, ns, K_SEG, c->Q.g, 0);
    fine(c, 12);
    LAUNCH_S(k_make_cands, ns, c->D, c->C, c->S, 0, ns, X, c->L, lmin2);
    fine(c, 13);
    g_prof[0] += now_s() - t0;
    double t1 = now_s();
    run_regions(c, 0, ns, 0);
    g_prof[1] += now_s() - t1;
    nbase = ns;
    R.ncand = ns;
  } else {
    int nf = sorted_records(c, 1, RF_ENC, RF_BLOCK | RF_SKIP, c->Q.g);
    if (nf > 0) {
      phase = 1;
      ensure_cands(c, nf + 64);
      LAUNCH(k_set_cands, nf, c->C, 0, nf, K_FACE, c->Q.g, 0);
      nbase = nf;
    } else {
      LAUNCH(k_flag_bad, c->hc.nt, c->D, c->B, c->Q.a);
      int nb = select_flagged(c, c->Q.a, c->hc.nt, c->Q.g);
      if (nb == 0) { R.phase = -1; return R; }
      phase = 2;
      ensure_cands(c, nb + 64);
      LAUNCH(k_set_cands, nb, c->C, 0, nb, K_TET, c->Q.g, 0);
      nbase = nb;
    }
    fine(c, 27);
    LAUNCH_S(k_make_cands, nbase, c->D, c->C, c->S, 0, nbase, X, c->L, lmin2);
    fine(c, 12);
    double t1 = now_s();
    // redirects first (refine.py:603-662): dropped candidates need no region
    grid_sync(c);
    LAUNCH(k_grid_cands, nbase, c->D, c->G, c->C, 0, nbase);
    fine(c, 28);
    CK(cudaMemsetAsync(c->d_int + 60, 0, 8, c->st));
    LAUNCH(k_redirect, nbase, c->D, c->C, 0, nbase, c->d_int + 60);
    fine(c, 13);
    ensure_tmp(c, nbase + 1);
    LAUNCH(k_kept, nbase, c->C, nbase, c->Q.a);
    int redir[2] = {0, 0};
    CK(cudaMemcpyAsync(redir, c->d_int + 60, 8, cudaMemcpyDeviceToHost, c->st));   // read with the scan below
    int kept = scan_total(c, c->Q.a, c->Q.b, nbase);
    LAUNCH(k_pool_pos, nbase, c->C, nbase, c->Q.b, c->Q.a);
    fine(c, 29);
    // only rounds with redirect hits pay for the flagged-record sorts
    int nrs = redir[0] > 0 ? append_redirects(c, 0, nbase, kept, X) : 0;
    int nrf = phase == 2 && redir[1] > 0 ? append_redirects(c, 1, nbase + nrs, kept + nrs, X) : 0;
    fine(c, 14);
    R.ncand = kept + nrs + nrf;
    g_prof[0] += now_s() - t0;
    t1 = now_s();
    nbase += nrs + nrf;
    run_regions(c, 0, nbase, 0);
    g_prof[1] += now_s() - t1;
    if (R.ncand == 0) { R.phase = -1; return R; }
  }
  int n = nbase;
  fine(c, 23);
  double t1 = now_s();
  ensure_tmp(c, n + 1);
  LAUNCH(k_states, n, c->C, n, c->Q.a, c->Q.b);
  int nok = scan_total(c, c->Q.a, c->Q.c, n);
  int nfail = select_flagged(c, c->Q.b, n, c->Q.h);
  fine(c, 15);
  rank_candidates(c, n);
  fine(c, 16);
  if (c->blast) run_filter_strict(c, n); else run_filter(c, n, nullptr);
  fine(c, 17);
  g_prof[2] += now_s() - t1;
  R.failed = nfail;
  R.phase = phase;
  insert_accepted(c, n, &R.acc, &R.inserted, round_no);
  R.rej = nok - R.acc;
  t1 = now_s();
  fine(c, -1);
  if (nfail > 0) {
    FallbackIO F; F.list = c->Q.h; F.n = nfail; F.round_no = round_no; F.seed = c->seed;
    F.with_facets = c->npoly > 0; F.lmin2 = lmin2; F.inserted = c->d_int + 20;
    CK(cudaMemsetAsync(c->d_int + 20, 0, 4, c->st));
    k_fallback<<<1, 1, 0, c->st>>>(c->D, c->C, c->SB, F, c->T, c->L);
    c->launches++;
    CK(cudaGetLastError());
    R.inserted += read_int(c, c->d_int + 20);
  }
  fine(c, 30);
  if (g_trace && phase == 2) {   // how many blasted tet candidates had their own tet taken by an accepted cavity
    CK(cudaMemsetAsync(c->d_int + 56, 0, 8, c->st));
    LAUNCH(k_count_seed_dead, n, c->D, c->C, n, c->d_int + 56);
    int h2[2];
    CK(cudaMemcpy(h2, c->d_int + 56, 8, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[seed] round %d rejected %d with dead seed tet %d\n", round_no, h2[0], h2[1]);
  }
  g_prof[5] += now_s() - t1;
  t1 = now_s();
  // post round: new vertices vs every constraint ball, then new / dirty
  // constraints vs the vertices around them
  fine(c, -1);
  grid_sync(c);
  fine(c, 7);
  if (c->hc.nv > c->reg_nv) LAUNCH(k_grid_newverts, c->hc.nv - c->reg_nv, c->D, c->G, c->reg_nv, c->hc.nv);
  c->reg_nv = c->hc.nv;
  fine(c, 8);
  CK(cudaMemsetAsync(c->d_int, 0, 16, c->st));
  LAUNCH_S(k_check, c->hc.nsegrec + c->hc.nfacerec, c->D, c->S, 0, c->d_int);
  if (R.inserted > 0) LAUNCH(k_clear_flag, c->hc.nsegrec + c->hc.nfacerec, c->D, RF_BLOCK);
  fine(c, 9);
  if (c->hc.nt > 4096) {
    ensure_tmp(c, c->hc.nt + 1);
    LAUNCH(k_compact_flags, c->hc.nt, c->D, c->tmpA);
    size_t need = 0;
    cub::DeviceReduce::Sum(nullptr, need, c->tmpA, c->d_int + 30, c->hc.nt, c->st);
    ensure_cub(c, need);
    cub::DeviceReduce::Sum(c->cub_tmp, need, c->tmpA, c->d_int + 30, c->hc.nt, c->st);
    int alive = read_int(c, c->d_int + 30);
    if ((long long)alive * 2 < c->hc.nt) compact_tets(c);
  }
  fine(c, 10);
  g_prof[6] += now_s() - t1;
  return R;
}

static void refine_impl(gq_ctx* c, const double* xyz, int n, int n_input, const int* seg, int m, const int* poff,
                        const int* pidx, int f, const int* keep, const int* order, const gq_config* cfg,
                        gq_counts* out) {
  c->B = cfg->B; c->max_rounds = cfg->max_rounds; c->seed = cfg->seed; c->verbose = cfg->flags & 1;
  c->blast = (cfg->flags & 2) != 0;
  g_fine = getenv("GQ_PROFILE") && atoi(getenv("GQ_PROFILE")) == 2;
  g_fine_ev = getenv("GQ_PROFILE") && atoi(getenv("GQ_PROFILE")) == 3;
  c->rpairs.clear(); c->fev.clear(); c->evused = 0;
  g_trace = getenv("GQ_TRACE") != nullptr;
  { int ws = getenv("GQ_WSTOP") ? atoi(getenv("GQ_WSTOP")) : 0; CK(cudaMemcpyToSymbol(g_wstop, &ws, 4)); }
  c->n_input = n_input; c->npoly = f;
  c->rounds.clear(); c->rtimes.clear(); c->launches = 0; c->region_ms = 0;
  free_all(c);
  unsigned int zero = 0;
  CK(cudaMemcpyToSymbol(g_err, &zero, 4));
  unsigned long long z4[4] = {0, 0, 0, 0};
  CK(cudaMemcpyToSymbol(g_exact_calls, z4, 32));
  unsigned long long z1 = 0;
  CK(cudaMemcpyToSymbol(g_region_calls, &z1, 8));
  CK(cudaMemcpyToSymbol(g_tested, &z1, 8));
  int npidx = f > 0 ? poff[f] : 0;
  double ta = now_s();
  alloc_mesh(c, n, m, f, npidx);
  CK(cudaDeviceSynchronize());
  if (getenv("GQ_PROFILE")) std::fprintf(stderr, "[gq] alloc %.1f ms\n", 1000 * (now_s() - ta));
  c->d_order = dmalloc<int>(n);
  Dev& D = c->D;
  // bbox / lmin (mesh.py:883-885, refine.py:532)
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = 0; i < n; ++i) for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], xyz[3 * i + k]); hi[k] = std::max(hi[k], xyz[3 * i + k]); }
  double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  double diag = std::sqrt(dx * dx + dy * dy + dz * dz);
  D.too_close_sq = 1e-24 * diag * diag;
  double lmin = 1e-4 * diag;
  D.lmin2 = lmin * lmin;
  CK(cudaMemcpyAsync(D.P, xyz, 24 * (size_t)n, cudaMemcpyHostToDevice, c->st));
  std::vector<uint8_t> org(n, 0);
  for (int i = n_input; i < n; ++i) org[i] = 1;
  CK(cudaMemcpyAsync(D.vorigin, org.data(), n, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(D.vert_tet, 0xff, 4 * (size_t)n, c->st));
  CK(cudaMemsetAsync(D.vsid, 0xff, 4 * (size_t)D.vcap, c->st));
  c->hc = Counters{};
  c->hc.nv = n;
  push(c);
  CK(cudaEventRecord(c->ev0, c->st));
  // polygon info
  c->polys.assign(m, {});
  std::vector<int> spo(m + 1, 0), sp;
  if (f > 0) {
    std::vector<std::pair<long long, int>> idx;
    std::vector<long long> keys(m);
    std::vector<int> sidx(m);
    for (int s = 0; s < m; ++s) {
      int u = std::min(seg[2 * s], seg[2 * s + 1]), v = std::max(seg[2 * s], seg[2 * s + 1]);
      idx.push_back({((long long)u << 32) | v, s});
    }
    std::sort(idx.begin(), idx.end());
    auto find_sid = [&](int a, int b) {
      long long k = ((long long)std::min(a, b) << 32) | std::max(a, b);
      auto it = std::lower_bound(idx.begin(), idx.end(), std::make_pair(k, -1));
      if (it == idx.end() || it->first != k) throw std::runtime_error("polygon edge not a segment");
      return it->second;
    };
    for (int pid = 0; pid < f; ++pid) {
      int o0 = poff[pid], o1 = poff[pid + 1], len = o1 - o0;
      for (int k = 0; k < len; ++k) {
        int a = pidx[o0 + k], b = pidx[o0 + (k + 1) % len];
        c->polys[find_sid(a, b)].push_back(pid);
      }
    }
    for (int s = 0; s < m; ++s) { spo[s + 1] = spo[s] + (int)c->polys[s].size(); for (int p : c->polys[s]) sp.push_back(p); }
    for (int s = 0; s < m; ++s) if (c->polys[s].size() > 4) throw std::runtime_error("segment shared by more than 4 polygons");
    CK(cudaMemcpy(D.poly_keep, keep, 8 * (size_t)f, cudaMemcpyHostToDevice));
    std::vector<uint8_t> obl(f, 1);
    for (int pid = 0; pid < f; ++pid)
      for (int k = 0; k < 3 && obl[pid]; ++k) {
        bool same = true;
        for (int q = poff[pid] + 1; q < poff[pid + 1] && same; ++q) same = xyz[3 * pidx[q] + k] == xyz[3 * pidx[poff[pid]] + k];
        if (same) obl[pid] = 0;
      }
    CK(cudaMemcpy(D.poly_obl, obl.data(), f, cudaMemcpyHostToDevice));
    if (!sp.empty()) CK(cudaMemcpy(D.segpoly, sp.data(), 4 * sp.size(), cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(D.segpoly_off, spo.data(), 4 * (size_t)(m + 1), cudaMemcpyHostToDevice));
  // init_delaunay
  init_delaunay(c, order, n);
  CK(cudaEventRecord(c->ev1, c->st));
  sync(c);
  float ims = 0; cudaEventElapsedTime(&ims, c->ev0, c->ev1); c->init_ms = ims;
  // constraints
  if (m > 0) {
    int* dseg = dmalloc<int>(2 * (size_t)m);
    CK(cudaMemcpy(dseg, seg, 8 * (size_t)m, cudaMemcpyHostToDevice));
    LAUNCH(k_segs_init, m, D, dseg, m);
    sync(c);
    dfree(dseg);
  }
  pull(c);
  c->hc.nsegrec = m;
  push(c);
  if (f > 0) {
    int* dpo = dmalloc<int>(f + 1); int* dpi = dmalloc<int>(std::max(npidx, 1));
    CK(cudaMemcpy(dpo, poff, 4 * (size_t)(f + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dpi, pidx, 4 * (size_t)npidx, cudaMemcpyHostToDevice));
    LAUNCH_S(k_facets_init, f, D, dpo, dpi, f, c->S, (int*)nullptr);
    sync(c);
    pull(c);
    LAUNCH(k_facets_records, c->hc.nt2, D, c->hc.nt2);
    sync(c);
    dfree(dpo); dfree(dpi);
  }
  LAUNCH(k_refresh_all, c->hc.nt, D);
  sync(c);
  for (int k = 0; k < 3; ++k) {
    c->G.lo[k] = lo[k];
    double ext = hi[k] - lo[k];
    c->G.inv[k] = ext > 0 ? c->G.G / ext : 0.0;
  }
  grid_sync(c);
  c->reg_nv = c->hc.nv;
  full_verify(c);
  // rounds (refine.py:866-925)
  int round_no = 0;
  while (round_no < c->max_rounds) {
    auto t0 = std::chrono::steady_clock::now();
    RoundOut R = run_round(c, round_no);
    if (R.phase < 0) {
      if (!full_verify(c)) break;
      round_no += 1;
      continue;
    }
    CK(cudaMemsetAsync(c->d_int + 4, 0, 16, c->st));
    pull(c);
    LAUNCH(k_count_pending, c->hc.nsegrec + c->hc.nfacerec, c->D, c->d_int + 4);
    int h[4];
    CK(cudaMemcpy(h, c->d_int + 4, 16, cudaMemcpyDeviceToHost));
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    c->rounds.push_back({round_no, R.phase, R.ncand, R.acc, R.rej, R.failed, R.inserted, h[2], h[3]});
    c->rtimes.push_back(dt);
    if (c->verbose)
      std::fprintf(stderr, "round %d phase=%d candidates=%lld accepted=%lld blasted=%lld failed=%lld inserted=%lld time=%.4f\n",
                   round_no, R.phase, R.ncand, R.acc, R.rej, R.failed, R.inserted, dt);
    round_no += 1;
  }
  CK(cudaEventRecord(c->ev1, c->st));
  sync(c);
  float ms = 0; cudaEventElapsedTime(&ms, c->ev0, c->ev1); c->dev_ms = ms;
  resolve_events(c);
  if (g_fine || g_fine_ev) {
    std::fprintf(stderr, "[gq fine]");
    for (int k = 0; k < 32; ++k) if (g_fine_t[k] > 0) { std::fprintf(stderr, " %s %.1f;", g_fine_names[k], 1000 * g_fine_t[k]); g_fine_t[k] = 0; }
    std::fprintf(stderr, "\n");
  }
  if (getenv("GQ_PROFILE")) {
    std::fprintf(stderr, "[gq profile] init %.1f ms (%d rounds);", c->init_ms, c->init_rounds);
    for (int k = 0; k < 8; ++k) { std::fprintf(stderr, " %s %.1f ms;", g_prof_names[k], 1000 * g_prof[k]); g_prof[k] = 0; }
    std::fprintf(stderr, " region kernels %.1f ms; launches %lld\n", c->region_ms, c->launches);
  }
  pull(c);
  if (out) {
    std::memset(out, 0, sizeof(*out));
    out->nv = c->hc.nv; out->nt = c->hc.nt;
    // live constraint counts
    std::vector<unsigned int> sf(c->hc.nsegrec), ff(c->hc.nfacerec);
    CK(cudaMemcpy(sf.data(), D.sg_fl, 4 * sf.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ff.data(), D.sf_fl, 4 * ff.size(), cudaMemcpyDeviceToHost));
    for (auto x : sf) out->n_subsegments += (x & RF_LIVE) ? 1 : 0;
    for (auto x : ff) out->n_subfaces += (x & RF_LIVE) ? 1 : 0;
    out->n_rounds = (int64_t)c->rounds.size();
    out->n_skipped = std::min(c->hc.nskip, c->L.cap);
    unsigned long long ex[4];
    CK(cudaMemcpyFromSymbol(ex, g_exact_calls, 32));
    for (int k = 0; k < 4; ++k) out->exact_calls[k] = (int64_t)ex[k];
    out->device_ms = c->dev_ms; out->init_ms = c->init_ms;
    out->kernel_launches = c->launches;
    unsigned long long rc = 0, tested = 0;
    CK(cudaMemcpyFromSymbol(&rc, g_region_calls, 8));
    CK(cudaMemcpyFromSymbol(&tested, g_tested, 8));
    out->region_calls = (int64_t)rc;
    out->region_ms = c->region_ms;
    std::vector<uint8_t> org2(c->hc.nv);
    CK(cudaMemcpy(org2.data(), D.vorigin, c->hc.nv, cudaMemcpyDeviceToHost));
    for (auto o : org2) { if (o) out->steiner_points++; else out->input_points++; }
    // 144 N_cand + 58 T_tested + 8 K_claims + 51 T_created + 1 T_deleted + 29 N_steiner
    long long ncand = 0, created = 0;
    for (auto& r : c->rounds) ncand += r[2];
    created = (long long)c->hc.nt;   // lower bound proxy (slots created since last compaction)
    long long steiner = c->hc.nv - n;
    (void)ncand; (void)created; (void)steiner;
    // region kernels' algorithmic bytes: 58 B per tet tested
    // (cavity + boundary neighbours: tv 16 + tn 16 + masks 2 + one vertex 24)
    // + 24 B per candidate point
    out->bytes_alg = 58 * (long long)tested + 24 * (long long)rc;
  }
}

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int gq_create(int device, gq_ctx** out) {
  if (!out) return GQ_EINVAL;
  gq_ctx* c = new gq_ctx();
  try {
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0)); CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreate(&c->er0)); CK(cudaEventCreate(&c->er1));
    CK(cudaDeviceSetLimit(cudaLimitStackSize, 16384));
    CK(cudaFuncSetAttribute(k_region_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BlockShared)));
    CK(cudaFuncSetAttribute(k_region_warp<WT1_MAXT, WT1_HASH, WT1_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(WR_WARPS * sizeof(WarpShared1))));
    if (WT1_MAXT != WT2_MAXT)
      CK(cudaFuncSetAttribute(k_region_warp<WT2_MAXT, WT2_HASH, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(WR_WARPS * sizeof(WarpShared2))));
    CK(cudaFuncSetAttribute(k_star_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(WS_WARPS * sizeof(StarShared))));
    CK(cudaFuncSetAttribute(k_init_stars_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(WS_WARPS * sizeof(StarShared))));
    CK(cudaFuncSetAttribute(k_init_region_warp<WT1_MAXT, WT1_HASH, WT1_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(WR_WARPS * sizeof(WarpShared1))));
    if (WT1_MAXT != WT2_MAXT)
      CK(cudaFuncSetAttribute(k_init_region_warp<WT2_MAXT, WT2_HASH, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(WR_WARPS * sizeof(WarpShared2))));
    CK(cudaFuncSetAttribute(k_init_region_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BlockShared)));
  } catch (std::exception& e) {
    c->err = e.what();
    *out = c;
    return GQ_ECUDA;
  }
  *out = c;
  return GQ_OK;
}

int gq_destroy(gq_ctx* c) {
  if (!c) return GQ_EINVAL;
  try {
    cudaSetDevice(c->device);
    free_all(c);
    for (cudaEvent_t e : c->evpool) cudaEventDestroy(e);
    { DevCache& C = dev_cache(); std::lock_guard<std::mutex> g(C.mu); cache_trim(C); }
    if (c->st) cudaStreamDestroy(c->st);
  } catch (...) {}
  delete c;
  return GQ_OK;
}

const char* gq_last_error(gq_ctx* c) { return c ? c->err.c_str() : "null context"; }

int gq_refine(gq_ctx* c, const double* xyz, int32_t n, int32_t n_input, const int32_t* seg, int32_t m,
              const int32_t* poly_off, const int32_t* poly_idx, int32_t f, const int32_t* poly_keep,
              const int32_t* order, const gq_config* cfg, gq_counts* counts) {
  if (!c || !xyz || n < 4 || !order || !cfg) return GQ_EINVAL;
  if (cfg->B <= 0 || cfg->max_rounds < 1) return GQ_EINVAL;
  try {
    CK(cudaSetDevice(c->device));
    refine_impl(c, xyz, n, n_input, seg, m, poly_off, poly_idx, f, poly_keep, order, cfg, counts);
  } catch (std::exception& e) {
    c->err = e.what();
    return std::string(e.what()).rfind("CUDA", 0) == 0 ? GQ_ECUDA : GQ_EDEVICE;
  }
  return GQ_OK;
}

int gq_export_mesh(gq_ctx* c, double* points, uint8_t* vert_origin, int32_t* vert_tet, int32_t* tv, int32_t* tn,
                   uint8_t* alive, uint8_t* sub_mask, uint8_t* seg_mask, double* ratio, uint8_t* skip_flag) {
  if (!c || !c->allocated) return GQ_EINVAL;
  try {
    pull(c);
    Dev& D = c->D;
    size_t nv = c->hc.nv, nt = c->hc.nt;
    if (points) CK(cudaMemcpy(points, D.P, 24 * nv, cudaMemcpyDeviceToHost));
    if (vert_origin) CK(cudaMemcpy(vert_origin, D.vorigin, nv, cudaMemcpyDeviceToHost));
    if (vert_tet) CK(cudaMemcpy(vert_tet, D.vert_tet, 4 * nv, cudaMemcpyDeviceToHost));
    if (tv) CK(cudaMemcpy(tv, D.tv, 16 * nt, cudaMemcpyDeviceToHost));
    if (tn) CK(cudaMemcpy(tn, D.tn, 16 * nt, cudaMemcpyDeviceToHost));
    if (alive) CK(cudaMemcpy(alive, D.alive, nt, cudaMemcpyDeviceToHost));
    if (sub_mask) CK(cudaMemcpy(sub_mask, D.sub, nt, cudaMemcpyDeviceToHost));
    if (seg_mask) CK(cudaMemcpy(seg_mask, D.seg, nt, cudaMemcpyDeviceToHost));
    if (ratio) CK(cudaMemcpy(ratio, D.ratio, 8 * nt, cudaMemcpyDeviceToHost));
    if (skip_flag) CK(cudaMemcpy(skip_flag, D.skip, nt, cudaMemcpyDeviceToHost));
  } catch (std::exception& e) { c->err = e.what(); return GQ_ECUDA; }
  return GQ_OK;
}

int gq_export_constraints(gq_ctx* c, int32_t* subsegments, int32_t* subfaces) {
  if (!c || !c->allocated) return GQ_EINVAL;
  try {
    pull(c);
    Dev& D = c->D;
    int ns = c->hc.nsegrec, nf = c->hc.nfacerec;
    std::vector<int2> uv(ns); std::vector<int> sid(ns); std::vector<unsigned int> sfl(ns);
    CK(cudaMemcpy(uv.data(), D.sg_uv, 8 * (size_t)ns, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sid.data(), D.sg_sid, 4 * (size_t)ns, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sfl.data(), D.sg_fl, 4 * (size_t)ns, cudaMemcpyDeviceToHost));
    std::vector<std::array<int, 3>> s;
    for (int r = 0; r < ns; ++r) if (sfl[r] & RF_LIVE) s.push_back({uv[r].x, uv[r].y, sid[r]});
    std::sort(s.begin(), s.end());
    if (subsegments) for (size_t i = 0; i < s.size(); ++i) for (int k = 0; k < 3; ++k) subsegments[3 * i + k] = s[i][k];
    std::vector<int4> fv(nf); std::vector<unsigned int> ffl(nf);
    CK(cudaMemcpy(fv.data(), D.sf_v, 16 * (size_t)nf, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ffl.data(), D.sf_fl, 4 * (size_t)nf, cudaMemcpyDeviceToHost));
    std::vector<std::array<int, 4>> fs;
    for (int r = 0; r < nf; ++r) if (ffl[r] & RF_LIVE) fs.push_back({fv[r].x, fv[r].y, fv[r].z, fv[r].w});
    std::sort(fs.begin(), fs.end());
    if (subfaces) for (size_t i = 0; i < fs.size(); ++i) for (int k = 0; k < 4; ++k) subfaces[4 * i + k] = fs[i][k];
  } catch (std::exception& e) { c->err = e.what(); return GQ_ECUDA; }
  return GQ_OK;
}

int gq_export_rounds(gq_ctx* c, int64_t* rows, double* seconds) {
  if (!c) return GQ_EINVAL;
  for (size_t i = 0; i < c->rounds.size(); ++i) {
    for (int k = 0; k < 9; ++k) rows[9 * i + k] = c->rounds[i][k];
    if (seconds) seconds[i] = c->rtimes[i];
  }
  return GQ_OK;
}

int gq_export_skipped(gq_ctx* c, int32_t* rows) {
  if (!c || !c->allocated) return GQ_EINVAL;
  try {
    pull(c);
    int n = std::min(c->hc.nskip, c->L.cap);
    std::vector<int> r(8 * (size_t)n);
    if (n) CK(cudaMemcpy(r.data(), c->L.rows, 32 * (size_t)n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
      rows[7 * i] = r[8 * i + 1]; rows[7 * i + 1] = r[8 * i + 2]; rows[7 * i + 2] = r[8 * i + 3];
      for (int k = 0; k < 4; ++k) rows[7 * i + 3 + k] = r[8 * i + 4 + k];
    }
  } catch (std::exception& e) { c->err = e.what(); return GQ_ECUDA; }
  return GQ_OK;
}

int gq_quality(gq_ctx* c, double B, int64_t* bad_count, int64_t* hist36) {
  if (!c || !c->allocated) return GQ_EINVAL;
  try {
    unsigned long long* d = dmalloc<unsigned long long>(37);
    CK(cudaMemset(d, 0, 37 * 8));
    pull(c);
    k_quality<<<grid_for(c->hc.nt), 128, 0, c->st>>>(c->D, B, d, d + 1);
    CK(cudaGetLastError());
    sync(c);
    unsigned long long h[37];
    CK(cudaMemcpy(h, d, 37 * 8, cudaMemcpyDeviceToHost));
    dfree(d);
    if (bad_count) *bad_count = (int64_t)h[0];
    if (hist36) for (int k = 0; k < 36; ++k) hist36[k] = (int64_t)h[1 + k];
  } catch (std::exception& e) { c->err = e.what(); return GQ_ECUDA; }
  return GQ_OK;
}

int gq_batch(int which, const double* in, int32_t n, int32_t width, int8_t* out8, double* outd) {
  try {
    double* din = dmalloc<double>((size_t)n * width);
    signed char* d8 = dmalloc<signed char>(n);
    double* dd = dmalloc<double>(4 * (size_t)n);
    unsigned int zero = 0;
    CK(cudaMemcpyToSymbol(g_err, &zero, 4));
    CK(cudaMemcpy(din, in, 8 * (size_t)n * width, cudaMemcpyHostToDevice));
    k_batch<<<grid_for(n), 128>>>(which, din, n, d8, dd);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (out8) CK(cudaMemcpy(out8, d8, n, cudaMemcpyDeviceToHost));
    if (outd) CK(cudaMemcpy(outd, dd, 32 * (size_t)n, cudaMemcpyDeviceToHost));
    dfree(din); dfree(d8); dfree(dd);
  } catch (std::exception&) { return GQ_ECUDA; }
  return GQ_OK;
}

}  // extern "C"
