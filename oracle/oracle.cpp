// TEST INFRASTRUCTURE ONLY -- the CPU oracle for gQM3D refinement.
//
// A sequential C++ restatement of the reference round driver
// /root/reference/pkg/src/tetrefine/refine.py:35-925 and its filter
// growblast.py:196-207 (greedy_oracle = the normative filter semantics,
// growblast.py:1-16).  It is imported only by tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg.  The product path
// (paper_1903_03406_b200) never links or calls it.
//
// Encroachment queries are exact and global, as the reference's
// ConstraintIndex / cKDTree scans are (refine.py:107-253, 314-335): the
// uniform grids below only enumerate candidates; every decision is the
// exact open-ball predicate of geom.hpp.
#include "oracle_facets.hpp"
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>

namespace orc {

static const uint64_t MASK64 = ~0ull;
inline uint64_t splitmix64(uint64_t x) {   // refine.py:35-39
  x = x + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Prio {
  int rank; uint64_t h; std::vector<int> canon;
  bool operator<(const Prio& o) const {
    if (rank != o.rank) return rank < o.rank;
    if (h != o.h) return h < o.h;
    return canon < o.canon;
  }
};
enum Kind { SEG = 0, FACE = 1, TET = 2 };

inline Prio make_priority(int kind, const std::vector<int>& canon, int round_no, uint64_t seed) {  // refine.py:45-52
  uint64_t h = splitmix64(seed ^ ((uint64_t)round_no * 0x9E3779B97F4A7C15ull));
  for (int v : canon) h = splitmix64(h ^ (uint64_t)((int64_t)v + 2));
  return Prio{kind, h, canon};
}

struct CK {
  int kind, a, b, c;   // 0 tet, 1 face, 2 subsegment
  bool operator==(const CK& o) const { return kind == o.kind && a == o.a && b == o.b && c == o.c; }
};
struct CKH { size_t operator()(const CK& k) const { return K3H()(K3{k.a ^ (k.kind << 29), k.b, k.c}); } };

struct Cand {
  int kind;
  int tet = -1;            // TET target
  uint64_t seg = 0;        // SEG target
  K3 face{0, 0, 0};        // FACE target
  double p[3];
  Prio prio;
  bool has_region = false;
  Region region;
  int seed = -1;           // walk seed (missing constraint)
  std::vector<int> allow_pids;  // allowed_cross = subfaces of these polygons
  bool has_extra = false;
  int sid = -1, pid = -1;
  std::string fail_reason;
};

struct Grid {
  double lo[3], h[3];
  int G = 1;
  void setup(const double* lo_, const double* hi_, int g) {
    G = std::max(1, g);
    for (int k = 0; k < 3; ++k) {
      lo[k] = lo_[k];
      double ext = hi_[k] - lo_[k];
      if (!(ext > 0)) ext = 1e-300;
      h[k] = ext / G;
    }
  }
  int ci(double x, int k) const {
    double f = (x - lo[k]) / h[k];
    if (!(f >= 0)) return 0;
    if (f >= G) return G - 1;
    return (int)f;
  }
  size_t cell(int i, int j, int k) const { return ((size_t)i * G + j) * G + k; }
};

struct Report {
  long long input_points = 0, steiner_points = 0, tet_count = 0, bad_tet_count = 0;
  std::vector<std::array<long long, 9>> per_round;  // round,phase,cands,acc,blasted,failed,inserted,pend_s,pend_f
  std::vector<double> round_time;
  std::vector<std::pair<int, std::vector<int>>> skipped_kind_verts;
  std::vector<int> skipped_reason;   // 0 degenerate 1 short_edge 2 too_close 3 cnss
  double total_time = 0, setup_time = 0;
  long long hist[36] = {0};
};

struct Driver {
  Mesh mesh;
  FacetComplex facets;
  bool has_facets = false;
  double B = 2.0;
  int max_rounds = 500;
  uint64_t seed = 0;
  double lmin = 0;
  std::set<uint64_t> enc_segs, blocked_segs;
  std::set<K3> enc_faces, blocked_faces;
  std::set<uint64_t> skipped_segs;
  std::set<K3> skipped_faces;
  Report rep;
  // per-round scratch
  std::vector<int> round_new_verts;
  std::vector<uint64_t> round_new_segs;
  std::vector<K3> round_new_faces;
  std::set<K3> round_dirty_faces;
  std::set<uint64_t> round_dirty_segs;
  // spatial enumeration
  double glo[3], ghi[3];
  Grid vg;
  std::vector<std::vector<int>> vcells;
  int vg_built_nv = 0;
  struct CRec { int kind; uint64_t seg; K3 face; double c[3]; double r2; bool live; };
  std::vector<CRec> crecs;
  std::unordered_map<uint64_t, int> seg_rec;
  std::unordered_map<K3, int, K3H> face_rec;
  Grid cg;
  std::vector<std::vector<int>> ccells;
  std::vector<int> cbig;

  bool skipped_seg(uint64_t k) const { return skipped_segs.count(k) > 0; }
  bool skipped_face(const K3& k) const { return skipped_faces.count(k) > 0; }

  // ---------------- spatial grids ----------------
  void rebuild_grids() {
    int g = (int)std::cbrt(std::max(1.0, mesh.nv / 4.0));
    g = std::min(std::max(g, 1), 160);
    vg.setup(glo, ghi, g);
    vcells.assign((size_t)g * g * g, {});
    for (int v = 0; v < mesh.nv; ++v) {
      const double* q = mesh.pt(v);
      vcells[vg.cell(vg.ci(q[0], 0), vg.ci(q[1], 1), vg.ci(q[2], 2))].push_back(v);
    }
    vg_built_nv = std::max(1, mesh.nv);
    cg.setup(glo, ghi, g);
    ccells.assign((size_t)g * g * g, {});
    cbig.clear();
    std::vector<CRec> old;
    old.swap(crecs);
    seg_rec.clear(); face_rec.clear();
    for (auto& r : old) if (r.live) register_crec(r);
  }
  void add_vertex_grid(int v) {
    if (mesh.nv > 2 * vg_built_nv) { rebuild_grids(); return; }
    const double* q = mesh.pt(v);
    vcells[vg.cell(vg.ci(q[0], 0), vg.ci(q[1], 1), vg.ci(q[2], 2))].push_back(v);
  }
  void register_crec(const CRec& r) {
    int id = (int)crecs.size();
    crecs.push_back(r);
    if (r.kind == SEG) seg_rec[r.seg] = id; else face_rec[r.face] = id;
    double rr = std::sqrt(r.r2) * (1.0 + 1e-9);
    int i0 = cg.ci(r.c[0] - rr, 0), i1 = cg.ci(r.c[0] + rr, 0);
    int j0 = cg.ci(r.c[1] - rr, 1), j1 = cg.ci(r.c[1] + rr, 1);
    int k0 = cg.ci(r.c[2] - rr, 2), k1 = cg.ci(r.c[2] + rr, 2);
    long long ncell = (long long)(i1 - i0 + 1) * (j1 - j0 + 1) * (k1 - k0 + 1);
    if (ncell > 64) { cbig.push_back(id); return; }
    for (int i = i0; i <= i1; ++i) for (int j = j0; j <= j1; ++j) for (int k = k0; k <= k1; ++k)
      ccells[cg.cell(i, j, k)].push_back(id);
  }
  void index_add_seg(uint64_t key) {   // refine.py:141-146
    if (seg_rec.count(key) && crecs[seg_rec[key]].live) return;
    const double *pu = mesh.pt(k2u(key)), *pv = mesh.pt(k2v(key));
    CRec r; r.kind = SEG; r.seg = key; r.live = true;
    for (int k = 0; k < 3; ++k) r.c[k] = (pu[k] + pv[k]) / 2.0;
    r.r2 = (pu[0] - r.c[0]) * (pu[0] - r.c[0]) + (pu[1] - r.c[1]) * (pu[1] - r.c[1]) + (pu[2] - r.c[2]) * (pu[2] - r.c[2]);
    register_crec(r);
  }
  void index_remove_seg(uint64_t key) { auto it = seg_rec.find(key); if (it != seg_rec.end()) { crecs[it->second].live = false; seg_rec.erase(it); } }
  void index_add_face(const K3& key) {
    if (face_rec.count(key) && crecs[face_rec[key]].live) return;
    Sphere s = circumcircle_tri(mesh.pt(key.a), mesh.pt(key.b), mesh.pt(key.c));
    CRec r; r.kind = FACE; r.face = key; r.live = true;
    for (int k = 0; k < 3; ++k) r.c[k] = s.c[k];
    r.r2 = s.r2;
    register_crec(r);
  }
  void index_remove_face(const K3& key) { auto it = face_rec.find(key); if (it != face_rec.end()) { crecs[it->second].live = false; face_rec.erase(it); } }

  // constraints whose open ball strictly contains p (exact)
  void encroached_by_point(const double* p, std::vector<uint64_t>* segs, std::vector<K3>* faces) {
    auto test = [&](int id) {
      CRec& r = crecs[id];
      if (!r.live) return;
      if (r.kind == SEG) {
        if (segs && encroaches_segment(mesh.pt(k2u(r.seg)), mesh.pt(k2v(r.seg)), p)) segs->push_back(r.seg);
      } else {
        if (faces && encroaches_face(mesh.pt(r.face.a), mesh.pt(r.face.b), mesh.pt(r.face.c), p)) faces->push_back(r.face);
      }
    };
    for (int id : ccells[cg.cell(cg.ci(p[0], 0), cg.ci(p[1], 1), cg.ci(p[2], 2))]) test(id);
    for (int id : cbig) test(id);
    if (segs) { std::sort(segs->begin(), segs->end()); segs->erase(std::unique(segs->begin(), segs->end()), segs->end()); }
    if (faces) { std::sort(faces->begin(), faces->end()); faces->erase(std::unique(faces->begin(), faces->end()), faces->end()); }
  }
  template <class F>
  bool any_vertex_in_ball(const double* c, double r, F pred) {
    double rr = r * (1.0 + 1e-9);
    int i0 = vg.ci(c[0] - rr, 0), i1 = vg.ci(c[0] + rr, 0);
    int j0 = vg.ci(c[1] - rr, 1), j1 = vg.ci(c[1] + rr, 1);
    int k0 = vg.ci(c[2] - rr, 2), k1 = vg.ci(c[2] + rr, 2);
    for (int i = i0; i <= i1; ++i) for (int j = j0; j <= j1; ++j) for (int k = k0; k <= k1; ++k)
      for (int v : vcells[vg.cell(i, j, k)]) if (pred(v)) return true;
    return false;
  }
  bool seg_encroached_scan(uint64_t key) {   // refine.py:314-323
    int u = k2u(key), v = k2v(key);
    const double *pu = mesh.pt(u), *pv = mesh.pt(v);
    double mid[3] = {(pu[0] + pv[0]) / 2.0, (pu[1] + pv[1]) / 2.0, (pu[2] + pv[2]) / 2.0};
    double r = std::sqrt(dist_sq(pu, pv)) / 2.0;
    return any_vertex_in_ball(mid, r, [&](int w) { return w != u && w != v && encroaches_segment(pu, pv, mesh.pt(w)); });
  }
  bool face_encroached_scan(const K3& key) {  // refine.py:326-335
    const double *a = mesh.pt(key.a), *b = mesh.pt(key.b), *c = mesh.pt(key.c);
    Sphere s = circumcircle_tri(a, b, c);
    return any_vertex_in_ball(s.c, std::sqrt(s.r2), [&](int w) {
      return w != key.a && w != key.b && w != key.c && encroaches_face(a, b, c, mesh.pt(w)); });
  }

  // ---------------- setup / verify ----------------
  void setup(const double* pts, int n, int n_input, const int* seg, int m, const int* poff, const int* pidx, int f,
             const int* order) {
    mesh.init_delaunay(pts, n, order);
    for (int v = n_input; v < n; ++v) mesh.origin[v] = 1;
    lmin = 1e-4 * mesh.bbox_diag;
    std::vector<double> P(pts, pts + 3 * (size_t)n);
    std::vector<std::array<int, 2>> segs;
    for (int i = 0; i < m; ++i) segs.push_back({seg[2 * i], seg[2 * i + 1]});
    std::vector<std::vector<int>> polys;
    for (int i = 0; i < f; ++i) polys.push_back(std::vector<int>(pidx + poff[i], pidx + poff[i + 1]));
    has_facets = f > 0;
    if (has_facets) facets.init(P, segs, polys);
    for (int sid = 0; sid < m; ++sid) mesh.subsegments[k2(segs[sid][0], segs[sid][1])] = sid;
    if (has_facets)
      for (size_t pid = 0; pid < polys.size(); ++pid)
        for (auto& key : facets.keys_by_pid[pid]) mesh.subfaces[key] = (int)pid;
    for (int t = 0; t < mesh.nt; ++t) if (mesh.alive[t]) mesh.refresh_masks(t);
    for (int k = 0; k < 3; ++k) { glo[k] = INFINITY; ghi[k] = -INFINITY; }
    for (int i = 0; i < n; ++i) for (int k = 0; k < 3; ++k) { glo[k] = std::min(glo[k], pts[3 * i + k]); ghi[k] = std::max(ghi[k], pts[3 * i + k]); }
    rebuild_grids();
    std::vector<uint64_t> sk; for (auto& kv : mesh.subsegments) sk.push_back(kv.first);
    std::sort(sk.begin(), sk.end());
    for (auto k : sk) index_add_seg(k);
    std::vector<K3> fk; for (auto& kv : mesh.subfaces) fk.push_back(kv.first);
    std::sort(fk.begin(), fk.end());
    for (auto& k : fk) index_add_face(k);
    full_verify();
  }

  bool full_verify() {   // refine.py:549-571
    bool found = false;
    std::vector<uint64_t> sk; for (auto& kv : mesh.subsegments) sk.push_back(kv.first);
    std::sort(sk.begin(), sk.end());
    for (auto key : sk) {
      if (skipped_seg(key) || enc_segs.count(key)) continue;
      if (!mesh.edge_exists(k2u(key), k2v(key)) || seg_encroached_scan(key)) { enc_segs.insert(key); found = true; }
    }
    std::vector<K3> fk; for (auto& kv : mesh.subfaces) fk.push_back(kv.first);
    std::sort(fk.begin(), fk.end());
    for (auto& key : fk) {
      if (skipped_face(key) || enc_faces.count(key)) continue;
      if (mesh.find_tet_with_face(key).first < 0 || face_encroached_scan(key)) { enc_faces.insert(key); found = true; }
    }
    blocked_segs.clear(); blocked_faces.clear();
    return found || !enc_segs.empty() || !enc_faces.empty();
  }

  // ---------------- candidates ----------------
  AllowFn allow_fn(const Cand& c) {
    if (c.allow_pids.empty()) return nullptr;
    std::vector<int> pids = c.allow_pids;
    Mesh* m = &mesh;
    return [m, pids](const K3& k) {
      auto it = m->subfaces.find(k);
      if (it == m->subfaces.end()) return false;
      for (int p : pids) if (p == it->second) return true;
      return false;
    };
  }

  int walk_seed(const double* p, int near_vertex) {   // refine.py:416-418
    int hint = mesh.vert_tet[near_vertex];
    return mesh.walk(p, hint >= 0 ? hint : -1);
  }

  Cand make_cand(int kind, int tet, uint64_t seg, const K3& face, int round_no, bool with_facets) {  // refine.py:338-375
    Cand c; c.kind = kind;
    if (kind == TET) {
      const int* q = &mesh.tv[4 * (size_t)tet];
      std::vector<int> canon(q, q + 4);
      std::sort(canon.begin(), canon.end());
      c.tet = tet;
      Sphere s = circumsphere_tet(mesh.pt(q[0]), mesh.pt(q[1]), mesh.pt(q[2]), mesh.pt(q[3]));
      c.p[0] = s.c[0]; c.p[1] = s.c[1]; c.p[2] = s.c[2];
      c.prio = make_priority(TET, canon, round_no, seed);
      return c;
    }
    if (kind == SEG) {
      c.seg = seg;
      int u = k2u(seg), v = k2v(seg);
      const double *pu = mesh.pt(u), *pv = mesh.pt(v);
      for (int k = 0; k < 3; ++k) c.p[k] = (pu[k] + pv[k]) / 2.0;
      c.prio = make_priority(SEG, {u, v}, round_no, seed);
      c.sid = mesh.subsegments.at(seg);
      if (!mesh.edge_exists(u, v)) c.seed = walk_seed(c.p, u);
    } else {
      c.face = face;
      Sphere s = circumcircle_tri(mesh.pt(face.a), mesh.pt(face.b), mesh.pt(face.c));
      c.p[0] = s.c[0]; c.p[1] = s.c[1]; c.p[2] = s.c[2];
      c.prio = make_priority(FACE, {face.a, face.b, face.c}, round_no, seed);
      c.pid = mesh.subfaces.at(face);
      if (mesh.find_tet_with_face(face).first < 0) c.seed = walk_seed(c.p, face.a);
    }
    if (with_facets) {
      if (kind == SEG) c.allow_pids = facets.segment_polygons[c.sid];
      else c.allow_pids = {c.pid};
      c.has_extra = true;
    }
    return c;
  }

  std::vector<int> seeds_for(Cand& c) {   // mesh.py:416-433
    if (c.seed >= 0) return {c.seed};
    if (c.kind == TET) return {c.tet};
    if (c.kind == SEG) {
      std::vector<int> ring = mesh.tets_around_edge(k2u(c.seg), k2v(c.seg));
      std::sort(ring.begin(), ring.end());
      if (ring.empty()) throw CNSS("subsegment not an edge");
      return ring;
    }
    auto ti = mesh.find_tet_with_face(c.face);
    if (ti.first < 0) throw CNSS("subface not a face");
    int u = mesh.nbt(ti.first, ti.second);
    std::vector<int> s{ti.first};
    if (u >= 0 && mesh.alive[u] && u != ti.first) s.push_back(u);
    std::sort(s.begin(), s.end());
    return s;
  }

  // refine.py:378-413
  bool obstructed_subface(int t, const double* c, K3* out) {
    int cur = t, prev = -1;
    int max_steps = mesh.walk_steps_cap(64);
    for (int step = 0; step < max_steps; ++step) {
      if (mesh.is_ghost(cur)) { K3 key = mesh.face_key(cur, 3); if (mesh.subfaces.count(key)) { *out = key; return true; } return false; }
      bool moved = false;
      for (int k = 0; k < 4; ++k) {
        int i = (k + step) & 3;
        int u = mesh.nbt(cur, i);
        if (u == prev) continue;
        int f[3]; mesh.face_verts(cur, i, f);
        if (orient3d(mesh.pt(f[0]), mesh.pt(f[1]), mesh.pt(f[2]), c) > 0) {
          if (mesh.is_ghost(u)) { K3 key = mesh.face_key(cur, i); if (mesh.subfaces.count(key)) { *out = key; return true; } return false; }
          prev = cur; cur = u; moved = true; break;
        }
      }
      if (!moved) return false;
    }
    int end = mesh.walk(c, t);
    if (mesh.is_ghost(end)) { K3 key = mesh.face_key(end, 3); if (mesh.subfaces.count(key)) { *out = key; return true; } }
    return false;
  }

  void record_skip(int kind, const std::vector<int>& canon, int reason) {
    rep.skipped_kind_verts.push_back({kind, canon});
    rep.skipped_reason.push_back(reason);
  }
  std::vector<int> tet_canon(int t) { const int* q = &mesh.tv[4 * (size_t)t]; std::vector<int> c(q, q + 4); std::sort(c.begin(), c.end()); return c; }

  // refine.py:583-665
  int build_pool(int round_no, std::vector<Cand>& pool) {
    std::vector<uint64_t> segs;
    for (auto k : enc_segs) if (!blocked_segs.count(k) && mesh.subsegments.count(k) && !skipped_seg(k)) segs.push_back(k);
    for (auto it = enc_segs.begin(); it != enc_segs.end();) { if (!mesh.subsegments.count(*it)) it = enc_segs.erase(it); else ++it; }
    std::sort(segs.begin(), segs.end(), [](uint64_t x, uint64_t y) { return std::make_pair(k2u(x), k2v(x)) < std::make_pair(k2u(y), k2v(y)); });
    if (!segs.empty()) {
      for (auto k : segs) pool.push_back(make_cand(SEG, -1, k, {}, round_no, has_facets));
      return SEG;
    }
    std::vector<K3> faces;
    for (auto& k : enc_faces) if (!blocked_faces.count(k) && mesh.subfaces.count(k) && !skipped_face(k)) faces.push_back(k);
    for (auto it = enc_faces.begin(); it != enc_faces.end();) { if (!mesh.subfaces.count(*it)) it = enc_faces.erase(it); else ++it; }
    if (!faces.empty()) {
      std::set<std::pair<int, int>> redirect;
      for (auto& k : faces) {
        Cand c = make_cand(FACE, -1, 0, k, round_no, has_facets);
        std::vector<uint64_t> hit;
        encroached_by_point(c.p, &hit, nullptr);
        bool any = false;
        for (auto h : hit) if (!skipped_seg(h)) { redirect.insert({k2u(h), k2v(h)}); any = true; }
        if (!any) pool.push_back(c);
      }
      for (auto& uv : redirect) pool.push_back(make_cand(SEG, -1, k2(uv.first, uv.second), {}, round_no, has_facets));
      return FACE;
    }
    std::vector<int> bad;
    for (int t = 0; t < mesh.nt; ++t)
      if (mesh.alive[t] == 1 && mesh.tv[4 * (size_t)t + 3] >= 0 && mesh.ratio[t] > B && mesh.skip_flag[t] == 0) bad.push_back(t);
    if (!bad.empty()) {
      std::set<std::pair<int, int>> rsegs;
      std::set<K3> rfaces;
      std::vector<Cand> cands;
      for (int t : bad) {
        Cand c;
        try { c = make_cand(TET, t, 0, {}, round_no, false); }
        catch (std::exception&) { mesh.skip_flag[t] = 1; record_skip(TET, tet_canon(t), 0); continue; }
        const int* q = &mesh.tv[4 * (size_t)t];
        double r2 = circumsphere_tet(mesh.pt(q[0]), mesh.pt(q[1]), mesh.pt(q[2]), mesh.pt(q[3])).r2;
        if (r2 < lmin * lmin) { mesh.skip_flag[t] = 1; record_skip(TET, tet_canon(t), 1); continue; }
        cands.push_back(std::move(c));
      }
      for (auto& c : cands) {
        std::vector<uint64_t> sh; std::vector<K3> fh;
        encroached_by_point(c.p, &sh, &fh);
        bool anys = false, anyf = false;
        for (auto h : sh) if (!skipped_seg(h)) anys = true;
        for (auto& h : fh) if (!skipped_face(h)) anyf = true;
        if (anys) { for (auto h : sh) if (!skipped_seg(h)) rsegs.insert({k2u(h), k2v(h)}); }
        else if (anyf) { for (auto& h : fh) if (!skipped_face(h)) rfaces.insert(h); }
        else {
          K3 hull;
          if (obstructed_subface(c.tet, c.p, &hull) && !skipped_face(hull)) rfaces.insert(hull);
          else pool.push_back(c);
        }
      }
      for (auto& uv : rsegs) { uint64_t k = k2(uv.first, uv.second); if (mesh.subsegments.count(k)) pool.push_back(make_cand(SEG, -1, k, {}, round_no, has_facets)); }
      for (auto& k : rfaces) if (mesh.subfaces.count(k)) pool.push_back(make_cand(FACE, -1, 0, k, round_no, has_facets));
      if (!pool.empty()) return TET;
    }
    return -1;
  }

  std::vector<CK> claim_keys(const Cand& c) {   // mesh.py:72-89 + growblast.py:67-72
    std::vector<CK> ks;
    const Region& R = c.region;
    for (int t : R.tets) ks.push_back({0, t, 0, 0});
    for (auto& k : R.bface_keys) ks.push_back({1, k.a, k.b, k.c});
    for (auto k : R.boundary_subsegments) ks.push_back({2, k2u(k), k2v(k), 0});
    for (auto k : R.enclosed_subsegments) ks.push_back({2, k2u(k), k2v(k), 0});
    for (auto& k : R.crossed_subfaces) ks.push_back({1, k.a, k.b, k.c});
    if (c.has_extra) {
      if (c.kind == SEG) ks.push_back({2, k2u(c.seg), k2v(c.seg), 0});
      else if (c.kind == FACE) ks.push_back({1, c.face.a, c.face.b, c.face.c});
    }
    return ks;
  }

  // growblast.py:123-193 with the greedy semantics of growblast.py:196-207
  void filter(std::vector<Cand>& pool, std::vector<int>& accepted, std::vector<int>& rejected, std::vector<int>& failed) {
    std::vector<int> ok;
    for (size_t i = 0; i < pool.size(); ++i) {
      Cand& c = pool[i];
      try {
        std::vector<int> seeds = seeds_for(c);
        c.region = mesh.delaunay_region(c.p, seeds, allow_fn(c));
        c.has_region = true;
      } catch (TooClose&) { c.fail_reason = "too_close"; failed.push_back((int)i); continue; }
      catch (CNSS&) { c.fail_reason = "cavity_not_star_shaped"; failed.push_back((int)i); continue; }
      if (c.region.min_vertex_dist_sq <= mesh.too_close_sq) { c.fail_reason = "too_close"; failed.push_back((int)i); continue; }
      ok.push_back((int)i);
    }
    std::vector<int> order = ok;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pool[a].prio < pool[b].prio; });
    std::unordered_set<CK, CKH> claimed;
    std::unordered_set<int> acc;
    for (int i : order) {
      auto ks = claim_keys(pool[i]);
      bool clash = false;
      for (auto& k : ks) if (claimed.count(k)) { clash = true; break; }
      if (clash) continue;
      for (auto& k : ks) claimed.insert(k);
      accepted.push_back(i);
      acc.insert(i);
    }
    for (int i : ok) if (!acc.count(i)) rejected.push_back(i);
  }

  std::map<int, std::vector<K3>> crossed_by_pid(const Region& R) {
    std::map<int, std::vector<K3>> out;
    for (auto& k : R.crossed_subfaces) {
      auto it = mesh.subfaces.find(k);
      if (it != mesh.subfaces.end()) out[it->second].push_back(k);
    }
    return out;
  }

  void apply_face_delta(const std::vector<K3>& rem, const std::vector<std::pair<K3, int>>& add) {
    for (auto& k : rem) { index_remove_face(k); enc_faces.erase(k); }
    for (auto& ka : add) { index_add_face(ka.first); round_new_faces.push_back(ka.first); round_dirty_faces.insert(ka.first); }
  }

  // refine.py:685-737
  int insert_candidate(Cand& c) {
    int vid_expected = mesh.nv;
    std::vector<K3> rem;
    std::vector<std::pair<K3, int>> add;
    int vid;
    if (c.kind == SEG) {
      if (has_facets) facets.split_segment(c.sid, c.seg, vid_expected, c.p, crossed_by_pid(c.region), rem, add);
      vid = mesh.insert_point(c.p, c.region, 1, &c.seg, rem, add);
      add_vertex_grid(vid);
      index_remove_seg(c.seg);
      enc_segs.erase(c.seg);
      int u = k2u(c.seg), v = k2v(c.seg);
      for (uint64_t ch : {k2(u, vid), k2(v, vid)}) { index_add_seg(ch); round_new_segs.push_back(ch); }
      // keys use the real vid
      apply_face_delta(rem, add);
    } else if (c.kind == FACE) {
      auto cb = crossed_by_pid(c.region);
      std::vector<K3> crossed;
      auto it = cb.find(c.pid);
      if (it != cb.end()) crossed = it->second;
      facets.split_facet(c.pid, vid_expected, c.p, crossed, rem, add);
      vid = mesh.insert_point(c.p, c.region, 1, nullptr, rem, add);
      add_vertex_grid(vid);
      apply_face_delta(rem, add);
    } else {
      vid = mesh.insert_point(c.p, c.region, 1, nullptr, {}, {});
      add_vertex_grid(vid);
    }
    if (c.kind != TET) {
      std::set<K3> crossed(c.region.crossed_subfaces.begin(), c.region.crossed_subfaces.end());
      for (auto& k : rem) {
        if (crossed.count(k)) continue;
        auto ti = mesh.find_tet_with_face(k);
        if (ti.first >= 0) {
          mesh.refresh_masks(ti.first);
          int u = mesh.nbt(ti.first, ti.second);
          if (u >= 0 && mesh.alive[u]) mesh.refresh_masks(u);
        }
      }
    }
    round_new_verts.push_back(vid);
    for (auto& k : c.region.boundary_subfaces) round_dirty_faces.insert(k);
    for (auto k : c.region.boundary_subsegments) round_dirty_segs.insert(k);
    return vid;
  }

  void skip_candidate(const Cand& c, int reason) {   // refine.py:801-812
    if (c.kind == TET) {
      int t = c.tet;
      if (t >= 0 && t < mesh.nt && mesh.alive[t]) { mesh.skip_flag[t] = 1; record_skip(TET, tet_canon(t), reason); }
    } else if (c.kind == SEG) {
      skipped_segs.insert(c.seg);
      record_skip(SEG, {k2u(c.seg), k2v(c.seg)}, reason);
      enc_segs.erase(c.seg);
    } else {
      skipped_faces.insert(c.face);
      record_skip(FACE, {c.face.a, c.face.b, c.face.c}, reason);
      enc_faces.erase(c.face);
    }
  }

  // refine.py:748-799
  bool fallback(const Cand& c, int round_no) {
    if (c.kind == TET && !(c.tet >= 0 && c.tet < mesh.nt && mesh.alive[c.tet])) return false;
    if (c.kind == SEG && !mesh.subsegments.count(c.seg)) return false;
    if (c.kind == FACE && !mesh.subfaces.count(c.face)) return false;
    try {
      Cand fresh = make_cand(c.kind, c.tet, c.seg, c.face, round_no, has_facets && c.kind != TET);
      if (c.kind == TET) {
        K3 hull;
        if (obstructed_subface(c.tet, fresh.p, &hull)) {
          if (mesh.subfaces.count(hull) && !skipped_face(hull)) enc_faces.insert(hull);
          return false;
        }
      }
      std::vector<int> seeds = seeds_for(fresh);
      fresh.region = mesh.delaunay_region(fresh.p, seeds, allow_fn(fresh));
      fresh.has_region = true;
      if (fresh.region.min_vertex_dist_sq <= mesh.too_close_sq) throw TooClose("fallback point coincides with a vertex");
      if (c.kind == TET && fresh.region.min_vertex_dist_sq < lmin * lmin) {
        mesh.skip_flag[c.tet] = 1; record_skip(TET, tet_canon(c.tet), 1);
        return false;
      }
      insert_candidate(fresh);
      return true;
    } catch (TooClose&) {
      skip_candidate(c, 2);
    } catch (CNSS& err) {
      if (!err.membrane_keys.empty()) {
        for (auto& mk : err.membrane_keys) if (mesh.subfaces.count(mk)) enc_faces.insert(mk);
        if (c.kind == SEG) blocked_segs.insert(c.seg);
        else if (c.kind == FACE) blocked_faces.insert(c.face);
      } else skip_candidate(c, 3);
    }
    return false;
  }

  // debug: compare the reference's global new-vertex query with the
  // mesh-local shortcut (constraints on the inserted cavities' boundaries)
  bool dbg_local = std::getenv("ORACLE_DEBUG_LOCAL") != nullptr;
  long long dbg_missed = 0;
  void post_round() {   // refine.py:816-858
    if (dbg_local) {
      for (int v : round_new_verts) {
        std::vector<uint64_t> s; std::vector<K3> fcs;
        encroached_by_point(mesh.pt(v), &s, &fcs);
        for (auto k : s) {
          if (skipped_seg(k) || enc_segs.count(k)) continue;
          bool covered = round_dirty_segs.count(k) || std::find(round_new_segs.begin(), round_new_segs.end(), k) != round_new_segs.end();
          if (!covered) { dbg_missed++; std::fprintf(stderr, "[local] new vertex %d encroaches non-dirty subsegment (%d,%d)\n", v, k2u(k), k2v(k)); }
        }
        for (auto& k : fcs) {
          if (skipped_face(k) || enc_faces.count(k)) continue;
          bool covered = round_dirty_faces.count(k) || std::find(round_new_faces.begin(), round_new_faces.end(), k) != round_new_faces.end();
          if (!covered) { dbg_missed++; std::fprintf(stderr, "[local] new vertex %d encroaches non-dirty subface (%d,%d,%d)\n", v, k.a, k.b, k.c); }
        }
      }
    }
    for (int v : round_new_verts) {
      std::vector<uint64_t> s; std::vector<K3> fcs;
      encroached_by_point(mesh.pt(v), &s, &fcs);
      for (auto k : s) if (!skipped_seg(k)) enc_segs.insert(k);
      for (auto& k : fcs) if (!skipped_face(k)) enc_faces.insert(k);
    }
    std::set<uint64_t> cs;
    for (auto k : round_new_segs) if (mesh.subsegments.count(k)) cs.insert(k);
    for (auto k : round_dirty_segs) if (mesh.subsegments.count(k)) cs.insert(k);
    std::set<K3> cf;
    for (auto& k : round_new_faces) if (mesh.subfaces.count(k)) cf.insert(k);
    for (auto& k : round_dirty_faces) if (mesh.subfaces.count(k)) cf.insert(k);
    if (dbg_local) {
      for (auto k : cs) {
        if (skipped_seg(k) || enc_segs.count(k)) continue;
        bool g = !mesh.edge_exists(k2u(k), k2v(k)) || seg_encroached_scan(k);
        bool l = false;
        auto ring = mesh.tets_around_edge(k2u(k), k2v(k));
        if (ring.empty()) l = true;
        for (int t : ring) for (int q = 0; q < 4; ++q) {
          int w = mesh.tv[4 * (size_t)t + q];
          if (w != GHOST && w != k2u(k) && w != k2v(k) && encroaches_segment(mesh.pt(k2u(k)), mesh.pt(k2v(k)), mesh.pt(w))) l = true;
        }
        if (g != l) { dbg_missed++; std::fprintf(stderr, "[local2] seg (%d,%d) global %d local %d\n", k2u(k), k2v(k), g, l); }
      }
      for (auto& k : cf) {
        if (skipped_face(k) || enc_faces.count(k)) continue;
        auto ti = mesh.find_tet_with_face(k);
        bool g = ti.first < 0 || face_encroached_scan(k);
        bool l = ti.first < 0;
        if (!l) {
          int w = mesh.tv[4 * (size_t)ti.first + ti.second];
          int u = mesh.nbt(ti.first, ti.second), j = (int)(mesh.tn[4 * (size_t)ti.first + ti.second] & 3);
          int w2 = mesh.tv[4 * (size_t)u + j];
          if (w != GHOST && encroaches_face(mesh.pt(k.a), mesh.pt(k.b), mesh.pt(k.c), mesh.pt(w))) l = true;
          if (w2 != GHOST && encroaches_face(mesh.pt(k.a), mesh.pt(k.b), mesh.pt(k.c), mesh.pt(w2))) l = true;
        }
        if (g != l) { dbg_missed++; std::fprintf(stderr, "[local2] face (%d,%d,%d) global %d local %d\n", k.a, k.b, k.c, g, l); }
      }
    }
    for (auto k : cs) {
      if (skipped_seg(k) || enc_segs.count(k)) continue;
      if (!mesh.edge_exists(k2u(k), k2v(k)) || seg_encroached_scan(k)) enc_segs.insert(k);
    }
    for (auto& k : cf) {
      if (skipped_face(k) || enc_faces.count(k)) continue;
      if (mesh.find_tet_with_face(k).first < 0 || face_encroached_scan(k)) enc_faces.insert(k);
    }
    if (!round_new_verts.empty()) { blocked_segs.clear(); blocked_faces.clear(); }
    if (mesh.nt > 4096) {
      long long a = 0;
      for (int t = 0; t < mesh.nt; ++t) a += mesh.alive[t] != 0;
      if (a * 2 < mesh.nt) mesh.compact();
    }
  }

  void run() {
    int round_no = 0;
    while (round_no < max_rounds) {
      std::vector<Cand> pool;
      int phase = build_pool(round_no, pool);
      if (phase < 0) {
        if (!full_verify()) break;
        round_no += 1;
        continue;
      }
      auto t0 = std::chrono::steady_clock::now();
      round_new_verts.clear(); round_new_segs.clear(); round_new_faces.clear();
      round_dirty_faces.clear(); round_dirty_segs.clear();
      std::vector<int> accepted, rejected, failed;
      filter(pool, accepted, rejected, failed);
      long long inserted = 0;
      for (int i : accepted) {
        Cand& c = pool[i];
        if (c.kind == TET && c.region.min_vertex_dist_sq < lmin * lmin) { skip_candidate(c, 1); continue; }
        insert_candidate(c);
        inserted++;
      }
      for (int i : failed) {
        Cand& c = pool[i];
        if (c.fail_reason == "too_close") skip_candidate(c, 2);
        else if (fallback(c, round_no)) inserted++;
      }
      post_round();
      double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      rep.per_round.push_back({round_no, phase, (long long)pool.size(), (long long)accepted.size(),
                               (long long)rejected.size(), (long long)failed.size(), inserted,
                               (long long)enc_segs.size(), (long long)enc_faces.size()});
      rep.round_time.push_back(dt);
      round_no += 1;
    }
  }
};

}  // namespace orc

using namespace orc;

extern "C" {

struct OrHandle { Driver d; int status = 0; char err[256] = {0}; };

// Refine an (already validated and box-augmented) PLC.  order = the numpy
// shuffle order of init_delaunay (mesh.py:878-880), computed by the caller.
void* or_refine(const double* pts, int n, int n_input, const int* seg, int m, const int* poff, const int* pidx,
                int f, const int* order, double B, int max_rounds, unsigned long long seed) {
  OrHandle* h = new OrHandle();
  try {
    auto t0 = std::chrono::steady_clock::now();
    h->d.B = B; h->d.max_rounds = max_rounds; h->d.seed = seed;
    h->d.setup(pts, n, n_input, seg, m, poff, pidx, f, order);
    h->d.rep.setup_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    h->d.run();
    h->d.rep.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } catch (std::exception& e) {
    h->status = 1;
    std::snprintf(h->err, sizeof(h->err), "%s", e.what());
  }
  return h;
}
int or_status(void* hp, char* buf, int n) { OrHandle* h = (OrHandle*)hp; std::snprintf(buf, n, "%s", h->err); return h->status; }
void or_free(void* hp) { delete (OrHandle*)hp; }

// counts: nv, nt, n_subsegs, n_subfaces, n_rounds, n_skipped, exact o3d, exact isp, region calls
void or_counts(void* hp, long long* out) {
  Driver& d = ((OrHandle*)hp)->d;
  out[0] = d.mesh.nv; out[1] = d.mesh.nt; out[2] = (long long)d.mesh.subsegments.size();
  out[3] = (long long)d.mesh.subfaces.size(); out[4] = (long long)d.rep.per_round.size();
  out[5] = (long long)d.rep.skipped_reason.size();
  out[6] = exact_stats().o3d; out[7] = exact_stats().isp; out[8] = d.mesh.region_calls;
}
void or_mesh(void* hp, double* pts, unsigned char* origin, int* vert_tet, int* tv, long long* tn, unsigned char* alive,
             unsigned char* sub_mask, unsigned char* seg_mask, double* ratio, unsigned char* skip) {
  Driver& d = ((OrHandle*)hp)->d;
  Mesh& m = d.mesh;
  std::memcpy(pts, m.P.data(), sizeof(double) * 3 * m.nv);
  std::memcpy(origin, m.origin.data(), m.nv);
  std::memcpy(vert_tet, m.vert_tet.data(), sizeof(int) * m.nv);
  std::memcpy(tv, m.tv.data(), sizeof(int) * 4 * (size_t)m.nt);
  std::memcpy(tn, m.tn.data(), sizeof(long long) * 4 * (size_t)m.nt);
  std::memcpy(alive, m.alive.data(), m.nt);
  std::memcpy(sub_mask, m.sub_mask.data(), m.nt);
  std::memcpy(seg_mask, m.seg_mask.data(), m.nt);
  std::memcpy(ratio, m.ratio.data(), sizeof(double) * m.nt);
  std::memcpy(skip, m.skip_flag.data(), m.nt);
}
// subsegments (u,v,sid) sorted; subfaces (a,b,c,pid) sorted
void or_constraints(void* hp, int* segs, int* faces) {
  Mesh& m = ((OrHandle*)hp)->d.mesh;
  std::vector<std::array<int, 3>> s;
  for (auto& kv : m.subsegments) s.push_back({k2u(kv.first), k2v(kv.first), kv.second});
  std::sort(s.begin(), s.end());
  for (size_t i = 0; i < s.size(); ++i) for (int k = 0; k < 3; ++k) segs[3 * i + k] = s[i][k];
  std::vector<std::array<int, 4>> f;
  for (auto& kv : m.subfaces) f.push_back({kv.first.a, kv.first.b, kv.first.c, kv.second});
  std::sort(f.begin(), f.end());
  for (size_t i = 0; i < f.size(); ++i) for (int k = 0; k < 4; ++k) faces[4 * i + k] = f[i][k];
}
void or_rounds(void* hp, long long* rows, double* times) {
  Report& r = ((OrHandle*)hp)->d.rep;
  for (size_t i = 0; i < r.per_round.size(); ++i) {
    for (int k = 0; k < 9; ++k) rows[9 * i + k] = r.per_round[i][k];
    times[i] = r.round_time[i];
  }
}
// skipped: kind, reason, nverts, v0..v3
void or_skipped(void* hp, int* rows) {
  Report& r = ((OrHandle*)hp)->d.rep;
  for (size_t i = 0; i < r.skipped_reason.size(); ++i) {
    int* q = rows + 7 * i;
    q[0] = r.skipped_kind_verts[i].first; q[1] = r.skipped_reason[i];
    q[2] = (int)r.skipped_kind_verts[i].second.size();
    for (int k = 0; k < 4; ++k) q[3 + k] = k < q[2] ? r.skipped_kind_verts[i].second[k] : -1;
  }
}
void or_times(void* hp, double* out) { Report& r = ((OrHandle*)hp)->d.rep; out[0] = r.setup_time; out[1] = r.total_time; }

// predicate entry points for the predicate parity tests (batched)
void or_orient3d(const double* p, int n, signed char* out) { for (int i = 0; i < n; ++i) out[i] = (signed char)orient3d(p + 12 * i, p + 12 * i + 3, p + 12 * i + 6, p + 12 * i + 9); }
void or_insphere(const double* p, int n, signed char* out) { for (int i = 0; i < n; ++i) out[i] = (signed char)insphere(p + 15 * i, p + 15 * i + 3, p + 15 * i + 6, p + 15 * i + 9, p + 15 * i + 12); }
void or_orient2d(const double* p, int n, signed char* out) { for (int i = 0; i < n; ++i) out[i] = (signed char)orient2d(p + 6 * i, p + 6 * i + 2, p + 6 * i + 4); }
void or_incircle2d(const double* p, int n, signed char* out) { for (int i = 0; i < n; ++i) out[i] = (signed char)incircle2d(p + 8 * i, p + 8 * i + 2, p + 8 * i + 4, p + 8 * i + 6); }
void or_incircle3d(const double* p, int n, signed char* out) {
  for (int i = 0; i < n; ++i) { try { out[i] = (signed char)incircle3d(p + 12 * i, p + 12 * i + 3, p + 12 * i + 6, p + 12 * i + 9); } catch (...) { out[i] = 99; } }
}
void or_encroach_seg(const double* p, int n, signed char* out) { for (int i = 0; i < n; ++i) out[i] = encroaches_segment(p + 9 * i, p + 9 * i + 3, p + 9 * i + 6); }
void or_encroach_face(const double* p, int n, signed char* out) {
  for (int i = 0; i < n; ++i) { try { out[i] = encroaches_face(p + 12 * i, p + 12 * i + 3, p + 12 * i + 6, p + 12 * i + 9); } catch (...) { out[i] = 99; } }
}
void or_circumsphere(const double* p, int n, double* out) {
  for (int i = 0; i < n; ++i) {
    try { Sphere s = circumsphere_tet(p + 12 * i, p + 12 * i + 3, p + 12 * i + 6, p + 12 * i + 9);
      out[4 * i] = s.c[0]; out[4 * i + 1] = s.c[1]; out[4 * i + 2] = s.c[2]; out[4 * i + 3] = s.r2; }
    catch (...) { for (int k = 0; k < 4; ++k) out[4 * i + k] = NAN; }
  }
}
void or_circumcircle(const double* p, int n, double* out) {
  for (int i = 0; i < n; ++i) {
    try { Sphere s = circumcircle_tri(p + 9 * i, p + 9 * i + 3, p + 9 * i + 6);
      out[4 * i] = s.c[0]; out[4 * i + 1] = s.c[1]; out[4 * i + 2] = s.c[2]; out[4 * i + 3] = s.r2; }
    catch (...) { for (int k = 0; k < 4; ++k) out[4 * i + k] = NAN; }
  }
}
}
