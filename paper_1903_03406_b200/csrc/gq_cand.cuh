// gq_cand.cuh -- candidate arrays, slabs, priorities, skip log and splitting points (refine.py:35-104, 338-375; mesh.py:416-433).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

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
#define MEMB_HUGE_OVF (-3)   // C.memb of a failed candidate whose cavity overflowed every region tier

// slab capacities (normal pass); overflowing candidates rerun with big slabs
#define CT 256
#define CF 576
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
  S.cancel = nullptr; S.me = 0;
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
  // huge slabs (bigi >= HUGE_BASE): capacities ht / hf / hc per slab, plus a
  // star pairing hash of hs slots per slab
  int* htets; int* hbf; int* hcr; int* hcrf; int* hbsub; int* hbseg; int* heseg;
  unsigned long long* hskey; int* hsv0; int* hsv1;
  int nhugecap, ht, hf, hc, hs;
  const int* segpoly;    // D.segpoly (allowed polygons of a segment shared by more than 4)
};
#define HUGE_BASE (1 << 28)
struct SlabView { int* tets; int* bf; int* cr; int* crf; int* bsub; int* bseg; int* eseg; int ct, cf, cc; };
__device__ __forceinline__ SlabView slab(const Cand& C, int c) {
  SlabView v;
  int b = C.bigi[c];
  if (b >= HUGE_BASE) {
    size_t h = (size_t)(b - HUGE_BASE);
    v.tets = C.htets + h * C.ht; v.bf = C.hbf + h * C.hf; v.cr = C.hcr + h * C.hc; v.crf = C.hcrf + h * C.hc;
    v.bsub = C.hbsub + h * C.hc; v.bseg = C.hbseg + h * C.hc; v.eseg = C.heseg + h * C.hc;
    v.ct = C.ht; v.cf = C.hf; v.cc = C.hc;
  } else if (b < 0) {
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
// 9 ints per row: round, kind, reason, n, v0..v3, order.  Rows are appended
// concurrently; `order` (stage << 28 | position: 0 candidate construction in
// pool order, 1 the accepted set in priority order, 2 the sequential fallback)
// restores the reference's recording order (refine.py:669-675) at export.
#define SKIP_ROW 9
struct SkipLog { int* rows; int cap; };
__device__ __forceinline__ int skip_order(int stage, int pos) { return (stage << 28) | (pos & ((1 << 28) - 1)); }
__device__ __noinline__ void log_skip(const Dev& D, const SkipLog& L, int round_no, int kind, int reason, const int* v, int n,
                                      int order) {
  atomicAdd(&D.ctr->skipr[(kind & 3) * 4 + (reason & 3)], 1u);
#ifdef GQ_DEBUG2D
  if (kind == K_SEG && n == 2) {
    const double *a = PT(D, v[0]), *b = PT(D, v[1]);
    double l = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]) + (a[2] - b[2]) * (a[2] - b[2]));
    printf("[skipseg] round %d reason %d len %.3e r %.6f %.6f z %.4f %.4f\n", round_no, reason, l,
           sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]), sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]), a[2], b[2]);
  }
#endif
  int k = atomicAdd(&D.ctr->nskip, 1);
  if (k >= L.cap) { raise_err(GQ_ERR_CAP); return; }
  int* r = L.rows + SKIP_ROW * (size_t)k;
  r[0] = round_no; r[1] = kind; r[2] = reason; r[3] = n;
  for (int i = 0; i < 4; ++i) r[4 + i] = i < n ? v[i] : -1;
  r[8] = order;
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

// Splitting point of subsegment record r: the midpoint (refine.py:91-104),
// except next to a small input angle.  Midpoint splitting of two segments
// meeting at < 45 degrees need not terminate (each split can make the other
// subsegment encroached again, down to rounding level: C4's torus quads have
// 18-degree corners); Shewchuk's concentric-shell rule splits a subsegment
// with exactly one such apex endpoint at the power of two nearest half its
// length, measured from the apex, so that subsegments around the apex come
// in equal lengths and stop encroaching each other.  Inputs without such an
// apex (every parity configuration: cube, random segments, rectangles,
// triangles with angles >= 50 degrees) split at the reference's midpoint;
// with one, the reference's own refinement has no termination guarantee.
__device__ __noinline__ void seg_split_point(const Dev& D, int r, double* p) {
  int2 e = D.sg_uv[r];
  const double *pu = PT(D, e.x), *pv = PT(D, e.y);
  int2 o = D.sid_uv[D.sg_sid[r]];
  bool au = (e.x == o.x || e.x == o.y) && D.vapex[e.x];
  bool av = (e.y == o.x || e.y == o.y) && D.vapex[e.y];
  if (au == av) {
    for (int k = 0; k < 3; ++k) p[k] = (pu[k] + pv[k]) / 2.0;
    return;
  }
  const double* a = au ? pu : pv;
  const double* b = au ? pv : pu;
  double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  double h = exp2(rint(log2(0.5 * len)));        // in [len/(2 sqrt 2), len/sqrt 2]
  double f = h / len;
  for (int k = 0; k < 3; ++k) p[k] = a[k] + d[k] * f;
}

// Convex-hull guard for constraint splits on an oblique hull (a PLC whose
// polygons tile a curved convex hull, C4's outer sphere: no box is added
// then, refine.py:462-475).  The ghost tets that close the mesh assume the
// hull stays convex; a midpoint / circumcentre rounded a few ulps INSIDE the
// hull faces it splits would leave a reflex hull edge, after which hull
// cavities stop starring and the hull subsegments split down to rounding
// level.  Such a point is pushed outward along the faces' normals by the
// smallest power-of-two step that puts it on or outside every hull face it
// splits (exact orient3d >= 0), so it becomes a hull vertex.  Axis-aligned
// hulls never need it: their split points round exactly onto the facet planes.
__device__ inline void hull_nudge(const Dev& D, double* p, const int4* hf, int nh) {
  bool ok = true;
  for (int k = 0; k < nh && ok; ++k) ok = orient3d(PT(D, hf[k].x), PT(D, hf[k].y), PT(D, hf[k].z), p) >= 0;
  if (ok) return;
  double N[3] = {0, 0, 0};
  for (int k = 0; k < nh; ++k) {
    const double *x = PT(D, hf[k].x), *y = PT(D, hf[k].y), *z = PT(D, hf[k].z);
    double u[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]}, v[3] = {z[0] - x[0], z[1] - x[1], z[2] - x[2]};
    double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    double l = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (l > 0) for (int a = 0; a < 3; ++a) N[a] += n[a] / l;
  }
  // steps are whole multiples of u = ulp(max |coordinate|): a coordinate moves
  // by 0 or by >= u, so no tiny coordinates appear (the exact predicates'
  // fixed-width integers size themselves by the exponent spread)
  double scale = fmax(fabs(p[0]), fmax(fabs(p[1]), fabs(p[2])));
  double u = ldexp(1.0, ilogb(scale) - 52);
  for (int e = 0; e < 40; ++e) {
    double step = ldexp(1.0, e);
    double q[3] = {p[0] + rint(N[0] * step) * u, p[1] + rint(N[1] * step) * u, p[2] + rint(N[2] * step) * u};
    bool good = true;
    for (int k = 0; k < nh && good; ++k) good = orient3d(PT(D, hf[k].x), PT(D, hf[k].y), PT(D, hf[k].z), q) >= 0;
    if (good) { p[0] = q[0]; p[1] = q[1]; p[2] = q[2]; return; }
  }
}
__device__ __noinline__ void hull_guard_seg(const Dev& D, int a, int b, double* p, Scratch& S) {
  int4 hf[8]; int nh = 0;
  around_vertex(D, a, S.tset, S.stack, 2 * S.cap, [&](int t) {
    int4 q = D.tv[t];
    if (q.w == GHOST && has_v(q, b) && nh < 8) hf[nh++] = q;
    return false;
  }, [&] { nh = 0; });
  if (nh) hull_nudge(D, p, hf, nh);
}
__device__ __noinline__ void hull_guard_face(const Dev& D, int slot, double* p) {
  if (slot < 0) return;
  int t = slot >> 2, u = tnk(D, t, slot & 3) >> 2;
  int4 hf[1];
  if (D.tv[t].w == GHOST) hf[0] = D.tv[t];
  else if (u >= 0 && D.tv[u].w == GHOST) hf[0] = D.tv[u];
  else return;
  hull_nudge(D, p, hf, 1);
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
    // A nearly flat tet can put its circumcentre at 1e40: far outside the hull,
    // where only the direction of the hull-exit walk matters (refine.py:378-413),
    // while the exact predicates' integers grow with the exponent spread.  Such a
    // point is pulled in along the same ray to 1000 bounding-box diagonals.
    {
      double diag = sqrt(D.lmin2) * 1e4, R = 1e3 * diag;
      const double *a = PT(D, q.x), *b = PT(D, q.y), *c3 = PT(D, q.z), *d = PT(D, q.w);
      double ctr[3], dv[3], l2 = 0;
      for (int k = 0; k < 3; ++k) { ctr[k] = 0.25 * (a[k] + b[k] + c3[k] + d[k]); dv[k] = p[k] - ctr[k]; l2 += dv[k] * dv[k]; }
      if (l2 > R * R) {
        double f = R / sqrt(l2);
        for (int k = 0; k < 3; ++k) p[k] = ctr[k] + dv[k] * f;
      }
    }
  } else if (kind == K_SEG) {
    int2 e = D.sg_uv[tgt];
    canon[0] = e.x; canon[1] = e.y; nc = 2;
    seg_split_point(D, tgt, p);
    if (X.with_facets && D.poly_obl_hull) hull_guard_seg(D, e.x, e.y, p, S);
    if (!edge_exists(D, e.x, e.y, S.tset, S.stack, 2 * S.cap)) C.seed[c] = walk_seed(D, p, e.x);
    if (X.with_facets) {
      int sid = D.sg_sid[tgt];
      int o0 = D.segpoly_off[sid], o1 = D.segpoly_off[sid + 1];
      int na = 0;
      int4 al = make_int4(-1, -1, -1, -1);
      if (o1 - o0 > 4) {          // more polygons than fit inline: refer to the segment's list
        al.x = o0; na = o1 - o0;
      } else {
        for (int o = o0; o < o1; ++o) {
          int pid = D.segpoly[o];
          if (na == 0) al.x = pid; else if (na == 1) al.y = pid; else if (na == 2) al.z = pid; else al.w = pid;
          ++na;
        }
      }
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
    if (D.poly_obl_hull && D.poly_obl[f.w]) hull_guard_face(D, slot, p);
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
  A.many = A.n > 4 ? C.segpoly + a.x : nullptr;   // a.x holds the offset into the segment's polygon list
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
    around_edge(D, e.x, e.y, S.tset, S.stack, 2 * S.cap, [&](int t) {
      if (n < 32) out[n++] = t;
      else { int mx = 0; for (int k = 1; k < 32; ++k) if (out[k] > out[mx]) mx = k; if (t < out[mx]) out[mx] = t; }
      return false;
    }, [&] { n = 0; });
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

