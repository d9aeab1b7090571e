// TEST INFRASTRUCTURE ONLY -- CPU oracle (see oracle/README.md).
//
// Sequential restatement of the reference triangulation
// (/root/reference/pkg/src/tetrefine/mesh.py and _kernels.py):
// flat arrays, ghost tets closing the hull, packed neighbours 4*t+f,
// Delaunay regions (grow / peel / seed component / finish), Bowyer-Watson
// starring, remembering walk, randomized incremental construction.
#pragma once
#include "geom.hpp"
#include <array>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <functional>
#include <map>
#include <set>
#include <cstdlib>

namespace orc {

static const int GHOST = -1;
static const int FACES[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};   // mesh.py:42
static const int EDGES[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}}; // mesh.py:43

struct K3 {
  int a, b, c;
  bool operator==(const K3& o) const { return a == o.a && b == o.b && c == o.c; }
  bool operator<(const K3& o) const {
    if (a != o.a) return a < o.a;
    if (b != o.b) return b < o.b;
    return c < o.c;
  }
};
struct K3H { size_t operator()(const K3& k) const {
  uint64_t h = (uint64_t)(uint32_t)k.a * 0x9E3779B97F4A7C15ull;
  h ^= (uint64_t)(uint32_t)k.b + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
  h ^= (uint64_t)(uint32_t)k.c * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
  return (size_t)h; } };
inline K3 sort3(int a, int b, int c) {
  if (a > b) std::swap(a, b);
  if (b > c) std::swap(b, c);
  if (a > b) std::swap(a, b);
  return K3{a, b, c};
}
inline uint64_t k2(int u, int v) {  // sorted pair key (u,v >= 0 in practice; ghost-safe)
  if (u > v) std::swap(u, v);
  return ((uint64_t)(uint32_t)(u + 1) << 32) | (uint32_t)(v + 1);
}
inline int k2u(uint64_t k) { return (int)(k >> 32) - 1; }
inline int k2v(uint64_t k) { return (int)(k & 0xffffffffu) - 1; }

struct CNSS : std::runtime_error {
  std::vector<K3> membrane_keys;
  CNSS(const char* m) : std::runtime_error(m) {}
};
struct TooClose : std::runtime_error { TooClose(const char* m) : std::runtime_error(m) {} };

struct Region {
  double p[3];
  std::vector<int> tets;                 // sorted
  std::vector<std::pair<int, int>> bfaces;
  std::vector<K3> bface_keys;
  std::vector<K3> crossed_subfaces, boundary_subfaces;   // sorted
  std::vector<uint64_t> boundary_subsegments, enclosed_subsegments;  // sorted
  double min_vertex_dist_sq = INFINITY;
};

// allowed_cross as a predicate over the current subface table (see refine.py:359-370)
using AllowFn = std::function<bool(const K3&)>;

struct Mesh {
  std::vector<double> P;           // 3*nv
  std::vector<uint8_t> origin;
  std::vector<int> vert_tet;
  int nv = 0;
  std::vector<int> tv;             // 4*cap
  std::vector<int64_t> tn;
  std::vector<uint8_t> alive, sub_mask, seg_mask, skip_flag;
  std::vector<double> ratio;
  int nt = 0;
  std::unordered_map<uint64_t, int> subsegments;   // sorted pair -> sid
  std::unordered_map<K3, int, K3H> subfaces;       // sorted triple -> pid
  double bbox_diag = 1.0, too_close_sq = 0.0;
  // scratch marks
  std::vector<uint32_t> mark, mark2;
  uint32_t epoch = 1, epoch2 = 1;
  long long region_calls = 0;

  const double* pt(int v) const { return &P[3 * (size_t)v]; }
  bool is_ghost(int t) const { return tv[4 * (size_t)t + 3] == GHOST; }

  void grow_tets(int need) {
    size_t cap = alive.size();
    if ((size_t)(nt + need) <= cap) return;
    size_t nc = std::max<size_t>(64, cap);
    while (nc < (size_t)(nt + need)) nc *= 2;
    tv.resize(4 * nc, 0);
    tn.resize(4 * nc, -1);
    alive.resize(nc, 0); sub_mask.resize(nc, 0); seg_mask.resize(nc, 0);
    skip_flag.resize(nc, 0); ratio.resize(nc, 0.0);
    mark.resize(nc, 0); mark2.resize(nc, 0);
  }
  int add_vertex(const double* p, int org) {
    P.push_back(p[0]); P.push_back(p[1]); P.push_back(p[2]);
    origin.push_back((uint8_t)org);
    vert_tet.push_back(-1);
    return nv++;
  }
  int new_tet(int a, int b, int c, int d) {
    grow_tets(1);
    int t = nt++;
    int* q = &tv[4 * (size_t)t];
    q[0] = a; q[1] = b; q[2] = c; q[3] = d;
    for (int k = 0; k < 4; ++k) tn[4 * (size_t)t + k] = -1;
    alive[t] = 1; sub_mask[t] = 0; seg_mask[t] = 0; skip_flag[t] = 0;
    for (int k = 0; k < 4; ++k) if (q[k] != GHOST) vert_tet[q[k]] = t;
    return t;
  }
  void set_bbox(const double* lo, const double* hi) {
    double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
    bbox_diag = std::sqrt(dx * dx + dy * dy + dz * dz);  // math.dist
    too_close_sq = 1e-24 * bbox_diag * bbox_diag;
  }
  void face_verts(int t, int i, int* f) const {
    const int* q = &tv[4 * (size_t)t];
    f[0] = q[FACES[i][0]]; f[1] = q[FACES[i][1]]; f[2] = q[FACES[i][2]];
  }
  K3 face_key(int t, int i) const { int f[3]; face_verts(t, i, f); return sort3(f[0], f[1], f[2]); }
  void set_nb(int t, int i, int u, int j) { tn[4 * (size_t)t + i] = 4 * (int64_t)u + j; tn[4 * (size_t)u + j] = 4 * (int64_t)t + i; }
  int nbt(int t, int i) const { return (int)(tn[4 * (size_t)t + i] >> 2); }
  bool has_v(int t, int v) const { const int* q = &tv[4 * (size_t)t]; return q[0] == v || q[1] == v || q[2] == v || q[3] == v; }

  // mesh.py:213-232
  void compute_ratio(int t) {
    if (is_ghost(t)) { ratio[t] = -1.0; return; }
    const int* q = &tv[4 * (size_t)t];
    const double *a = pt(q[0]), *b = pt(q[1]), *c = pt(q[2]), *d = pt(q[3]);
    Sphere s;
    try { s = circumsphere_tet(a, b, c, d); } catch (DegenerateTet&) { ratio[t] = INFINITY; return; }
    auto sq = [](const double* x, const double* y) {
      double e0 = x[0] - y[0], e1 = x[1] - y[1], e2 = x[2] - y[2];
      return e0 * e0 + e1 * e1 + e2 * e2; };
    double sh = sq(a, b);
    sh = std::min(sh, sq(a, c)); sh = std::min(sh, sq(a, d));
    sh = std::min(sh, sq(b, c)); sh = std::min(sh, sq(b, d)); sh = std::min(sh, sq(c, d));
    ratio[t] = std::sqrt(s.r2 / sh);
  }

  // mesh.py:236-262 (including the vert_tet side effect)
  std::vector<int> tets_around_vertex(int v) {
    int start = vert_tet[v];
    if (start < 0 || !alive[start] || !has_v(start, v)) {
      start = -1;
      for (int t = 0; t < nt; ++t) if (alive[t] && has_v(t, v)) { start = t; break; }
      if (start < 0) return {};
      vert_tet[v] = start;
    }
    std::vector<int> out{start};
    std::unordered_set<int> seen{start};
    std::vector<int> stack{start};
    while (!stack.empty()) {
      int t = stack.back(); stack.pop_back();
      const int* q = &tv[4 * (size_t)t];
      int local = 0;
      while (q[local] != v) ++local;
      for (int i = 0; i < 4; ++i) {
        if (i == local) continue;
        int u = nbt(t, i);
        if (u >= 0 && !seen.count(u) && alive[u]) { seen.insert(u); out.push_back(u); stack.push_back(u); }
      }
    }
    return out;
  }
  bool edge_exists(int u, int v) {
    for (int t : tets_around_vertex(u)) if (has_v(t, v)) return true;
    return false;
  }
  std::vector<int> tets_around_edge(int u, int v) {
    std::vector<int> r;
    for (int t : tets_around_vertex(u)) if (has_v(t, v)) r.push_back(t);
    return r;
  }
  std::pair<int, int> find_tet_with_face(const K3& key) {
    for (int t : tets_around_vertex(key.a)) {
      if (has_v(t, key.b) && has_v(t, key.c)) {
        for (int i = 0; i < 4; ++i) if (face_key(t, i) == key) return {t, i};
      }
    }
    return {-1, -1};
  }

  int hint_tet(int hint) {
    if (hint >= 0 && hint < nt && alive[hint] && !is_ghost(hint)) return hint;
    for (int t = 0; t < nt; ++t) if (alive[t] && !is_ghost(t)) return t;
    throw CNSS("mesh has no alive real tets");
  }

  int walk_steps_cap(int extra) const {
    double ntd = std::max(1.0, (double)nt);
    return (int)(10.0 * std::pow(ntd, 1.0 / 3.0)) + extra;
  }

  // mesh.py:322-371 (the numba walk makes the same decisions)
  int walk(const double* p, int hint) {
    int t = hint_tet(hint);
    int max_steps = walk_steps_cap(32);
    int step = 0, prev = -1;
    while (step < max_steps) {
      step += 1;
      if (is_ghost(t)) return t;
      bool moved = false;
      for (int k = 0; k < 4; ++k) {
        int i = (k + step) & 3;
        int u = nbt(t, i);
        if (u == prev) continue;
        int f[3]; face_verts(t, i, f);
        if (orient3d(pt(f[0]), pt(f[1]), pt(f[2]), p) > 0) { prev = t; t = u; moved = true; break; }
      }
      if (!moved) return t;
    }
    for (int s = 0; s < nt; ++s) {
      if (!alive[s] || is_ghost(s)) continue;
      bool in = true;
      for (int i = 0; i < 4 && in; ++i) {
        int f[3]; face_verts(s, i, f);
        if (orient3d(pt(f[0]), pt(f[1]), pt(f[2]), p) > 0) in = false;
      }
      if (in) return s;
    }
    for (int s = 0; s < nt; ++s) {
      if (alive[s] && is_ghost(s)) {
        const int* q = &tv[4 * (size_t)s];
        if (orient3d(pt(q[0]), pt(q[1]), pt(q[2]), p) > 0) return s;
      }
    }
    throw CNSS("walk failed to locate point");
  }

  // mesh.py:395-414
  bool in_region(int t, const double* p, const AllowFn& allowed) const {
    const int* q = &tv[4 * (size_t)t];
    if (q[3] == GHOST) {
      const double *a = pt(q[0]), *b = pt(q[1]), *c = pt(q[2]);
      int s = orient3d(a, b, c, p);
      if (s > 0) return true;
      if (s == 0) return incircle3d(a, b, c, p) > 0;
      if (allowed && allowed(face_key(t, 3))) return incircle3d(a, b, c, p) > 0;
      return false;
    }
    return insphere(pt(q[0]), pt(q[1]), pt(q[2]), pt(q[3]), p) > 0;
  }

  bool blocked(int t, int i, const AllowFn& allowed) const {
    if (!(sub_mask[t] & (1 << i))) return false;
    return !(allowed && allowed(face_key(t, i)));
  }

  // mesh.py:450-521 with the kernel's decision sequence (_kernels.py:392-635)
  Region delaunay_region(const double* p, const std::vector<int>& cands_in, const AllowFn& allowed) {
    region_calls++;
    std::vector<int> cands = cands_in;
    bool walked = false;
    int seed = -1;
    while (true) {
      seed = -1;
      for (int t : cands) {
        if (t < 0 || !alive[t]) continue;
        if (in_region(t, p, allowed)) { seed = t; break; }
      }
      if (seed >= 0) break;
      if (walked) throw CNSS("seed not in region");
      walked = true;
      int t = walk(p, cands.empty() ? -1 : cands[0]);
      cands = {t};
    }
    // grow (DFS)
    uint32_t ep = ++epoch;
    std::vector<int> cav{seed};
    mark[seed] = ep;
    std::vector<int> stack{seed};
    while (!stack.empty()) {
      int t = stack.back(); stack.pop_back();
      for (int i = 0; i < 4; ++i) {
        int u = nbt(t, i);
        if (u < 0 || mark[u] == ep || !alive[u]) continue;
        if (blocked(t, i, allowed)) continue;
        if (in_region(u, p, allowed)) { mark[u] = ep; cav.push_back(u); stack.push_back(u); }
      }
    }
    // shrink / seed component (confluent)
    while (true) {
      bool changed = true;
      while (changed) {
        changed = false;
        std::vector<int> snap;
        for (int t : cav) if (mark[t] == ep) snap.push_back(t);
        for (int t : snap) {
          if (mark[t] != ep) continue;
          for (int i = 0; i < 4; ++i) {
            int u = nbt(t, i);
            bool blk = blocked(t, i, allowed);
            if (mark[u] == ep && !blk) continue;
            int f[3]; face_verts(t, i, f);
            if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) continue;
            if (orient3d(pt(f[0]), pt(f[1]), pt(f[2]), p) >= 0) { mark[t] = 0; changed = true; break; }
          }
        }
        if (mark[seed] != ep) throw CNSS("seed shrunk away");
      }
      std::vector<int> live;
      for (int t : cav) if (mark[t] == ep) live.push_back(t);
      uint32_t e2 = ++epoch2;
      std::vector<int> comp{seed};
      mark2[seed] = e2;
      stack.assign(1, seed);
      while (!stack.empty()) {
        int t = stack.back(); stack.pop_back();
        for (int i = 0; i < 4; ++i) {
          int u = nbt(t, i);
          if (mark[u] != ep || mark2[u] == e2) continue;
          if (blocked(t, i, allowed)) continue;
          mark2[u] = e2; comp.push_back(u); stack.push_back(u);
        }
      }
      if (comp.size() == live.size()) { cav = live; break; }
      for (int t : live) if (mark2[t] != e2) mark[t] = 0;
      cav = comp;
    }
    // finish
    Region R;
    R.p[0] = p[0]; R.p[1] = p[1]; R.p[2] = p[2];
    std::sort(cav.begin(), cav.end());
    R.tets = cav;
    std::unordered_set<int> bverts;
    std::unordered_set<uint64_t> bedges;
    std::set<K3> seen_sub;
    std::set<uint64_t> seen_seg;
    for (int t : cav) {
      for (int i = 0; i < 4; ++i) {
        int u = nbt(t, i);
        bool blk = blocked(t, i, allowed);
        bool uin = mark[u] == ep;
        if (uin && !blk) continue;
        if (uin && blk) {
          CNSS e("constrained membrane face");
          e.membrane_keys.push_back(face_key(t, i));
          throw e;
        }
        int f[3]; face_verts(t, i, f);
        R.bfaces.push_back({t, i});
        R.bface_keys.push_back(sort3(f[0], f[1], f[2]));
        for (int k = 0; k < 3; ++k) if (f[k] != GHOST) bverts.insert(f[k]);
        if (f[0] != GHOST && f[1] != GHOST) bedges.insert(k2(f[0], f[1]));
        if (f[0] != GHOST && f[2] != GHOST) bedges.insert(k2(f[0], f[2]));
        if (f[1] != GHOST && f[2] != GHOST) bedges.insert(k2(f[1], f[2]));
      }
      int sm = sub_mask[t];
      if (sm) {
        for (int i = 0; i < 4; ++i) {
          if (!(sm & (1 << i))) continue;
          K3 key = face_key(t, i);
          if (seen_sub.count(key)) continue;
          seen_sub.insert(key);
          int u = nbt(t, i);
          bool crossed = (mark[u] == ep) && allowed && allowed(key);
          (crossed ? R.crossed_subfaces : R.boundary_subfaces).push_back(key);
        }
      }
      int em = seg_mask[t];
      if (em) {
        const int* q = &tv[4 * (size_t)t];
        for (int i = 0; i < 6; ++i) {
          if (!(em & (1 << i))) continue;
          uint64_t key = k2(q[EDGES[i][0]], q[EDGES[i][1]]);
          if (seen_seg.count(key)) continue;
          seen_seg.insert(key);
          (bedges.count(key) ? R.boundary_subsegments : R.enclosed_subsegments).push_back(key);
        }
      }
    }
    // NOTE: like region_kernel (_kernels.py:603-618) a subsegment is classified
    // when first met, against the boundary edges collected so far.
    std::sort(R.crossed_subfaces.begin(), R.crossed_subfaces.end());
    std::sort(R.boundary_subfaces.begin(), R.boundary_subfaces.end());
    std::sort(R.boundary_subsegments.begin(), R.boundary_subsegments.end(), [](uint64_t x, uint64_t y) {
      return std::make_pair(k2u(x), k2v(x)) < std::make_pair(k2u(y), k2v(y)); });
    std::sort(R.enclosed_subsegments.begin(), R.enclosed_subsegments.end(), [](uint64_t x, uint64_t y) {
      return std::make_pair(k2u(x), k2v(x)) < std::make_pair(k2u(y), k2v(y)); });
    for (int v : bverts) {
      const double* q = pt(v);
      double d = (q[0] - p[0]) * (q[0] - p[0]) + (q[1] - p[1]) * (q[1] - p[1]) + (q[2] - p[2]) * (q[2] - p[2]);
      if (d < R.min_vertex_dist_sq) R.min_vertex_dist_sq = d;
    }
    for (int t : cav) {
      const int* q = &tv[4 * (size_t)t];
      for (int k = 0; k < 4; ++k) if (q[k] != GHOST && !bverts.count(q[k])) throw CNSS("cavity swallows a vertex");
    }
    return R;
  }

  // mesh.py:827-840
  void refresh_masks(int t) {
    int sm = 0;
    for (int i = 0; i < 4; ++i) if (subfaces.count(face_key(t, i))) sm |= 1 << i;
    sub_mask[t] = (uint8_t)sm;
    int em = 0;
    const int* q = &tv[4 * (size_t)t];
    for (int i = 0; i < 6; ++i) {
      int a = q[EDGES[i][0]], b = q[EDGES[i][1]];
      if (a != GHOST && b != GHOST && subsegments.count(k2(a, b))) em |= 1 << i;
    }
    seg_mask[t] = (uint8_t)em;
  }

  // mesh.py:697-771 + _kernels.py:641-807
  int insert_point(const double* p, const Region& R, int org, const uint64_t* split_edge,
                   const std::vector<K3>& sub_removed, const std::vector<std::pair<K3, int>>& sub_added, int vid = -1) {
    if (R.min_vertex_dist_sq <= too_close_sq) throw TooClose("insertion point coincides with a vertex");
    if (vid < 0) vid = add_vertex(p, org);
    for (int t : R.tets) alive[t] = 0;
    std::vector<uint64_t> vid_segs;
    if (split_edge) {
      int u = k2u(*split_edge), v = k2v(*split_edge);
      auto it = subsegments.find(*split_edge);
      int parent = it->second;
      subsegments.erase(it);
      vid_segs = {k2(u, vid), k2(v, vid)};
      for (auto k : vid_segs) subsegments[k] = parent;
    }
    for (auto& k : sub_removed) subfaces.erase(k);
    std::vector<K3> added_keys;
    for (auto& kp : sub_added) {
      const K3& k = kp.first;
      K3 key = sort3(k.a == -1 ? vid : k.a, k.b == -1 ? vid : k.b, k.c == -1 ? vid : k.c);
      subfaces[key] = kp.second;
      added_keys.push_back(key);
    }
    // star kernel
    int nbf = (int)R.bfaces.size();
    grow_tets(nbf);
    std::unordered_set<K3, K3H> sub_keys(added_keys.begin(), added_keys.end());
    std::unordered_set<uint64_t> seg_keys(vid_segs.begin(), vid_segs.end());
    for (auto& key : R.bface_keys) {
      if (subfaces.count(key)) sub_keys.insert(key);
      int kk[3] = {key.a, key.b, key.c};
      int pr[3][2] = {{kk[0], kk[1]}, {kk[0], kk[2]}, {kk[1], kk[2]}};
      for (auto& e : pr) if (e[0] != GHOST && subsegments.count(k2(e[0], e[1]))) seg_keys.insert(k2(e[0], e[1]));
    }
    int nt0 = nt;
    for (int k = 0; k < nbf; ++k) {
      int t = R.bfaces[k].first, i = R.bfaces[k].second;
      int64_t packed = tn[4 * (size_t)t + i];
      int u = (int)(packed >> 2), j = (int)(packed & 3);
      int f[3]; face_verts(u, j, f);
      int ntt = nt0 + k;
      int* q = &tv[4 * (size_t)ntt];
      if (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) {
        int e0, e1;
        if (f[0] == GHOST) { e0 = f[1]; e1 = f[2]; }
        else if (f[1] == GHOST) { e0 = f[2]; e1 = f[0]; }
        else { e0 = f[0]; e1 = f[1]; }
        q[0] = e1; q[1] = e0; q[2] = vid; q[3] = GHOST;
      } else {
        q[0] = f[0]; q[1] = f[1]; q[2] = f[2]; q[3] = vid;
      }
      for (int m = 0; m < 4; ++m) {
        tn[4 * (size_t)ntt + m] = -1;
        if (q[m] != GHOST) vert_tet[q[m]] = ntt;
      }
      alive[ntt] = 1; sub_mask[ntt] = 0; seg_mask[ntt] = 0; skip_flag[ntt] = 0;
      K3 key = sort3(f[0], f[1], f[2]);
      int outer = -1;
      for (int m = 0; m < 4; ++m) {
        int g[3];
        const int* qq = q;
        g[0] = qq[FACES[m][0]]; g[1] = qq[FACES[m][1]]; g[2] = qq[FACES[m][2]];
        if (sort3(g[0], g[1], g[2]) == key) { outer = m; break; }
      }
      if (outer < 0) throw CNSS("unmatched faces after starring");
      tn[4 * (size_t)ntt + outer] = 4 * (int64_t)u + j;
      tn[4 * (size_t)u + j] = 4 * (int64_t)ntt + outer;
    }
    nt = nt0 + nbf;
    std::unordered_map<K3, int64_t, K3H> fmap;
    for (int k = 0; k < nbf; ++k) {
      int ntt = nt0 + k;
      for (int i = 0; i < 4; ++i) {
        int64_t pk = tn[4 * (size_t)ntt + i];
        if (pk >= 0 && alive[pk >> 2]) continue;
        K3 key = face_key(ntt, i);
        auto it = fmap.find(key);
        if (it != fmap.end()) {
          int64_t other = it->second;
          fmap.erase(it);
          tn[4 * (size_t)ntt + i] = other;
          tn[4 * (size_t)(other >> 2) + (other & 3)] = 4 * (int64_t)ntt + i;
        } else fmap[key] = 4 * (int64_t)ntt + i;
      }
    }
    if (!fmap.empty()) throw CNSS("unmatched faces after starring");
    for (int k = 0; k < nbf; ++k) {
      int ntt = nt0 + k;
      const int* q = &tv[4 * (size_t)ntt];
      int sm = 0;
      for (int i = 0; i < 4; ++i) {
        int g0 = q[FACES[i][0]], g1 = q[FACES[i][1]], g2 = q[FACES[i][2]];
        if (g0 != GHOST && g1 != GHOST && g2 != GHOST && sub_keys.count(sort3(g0, g1, g2))) sm |= 1 << i;
      }
      sub_mask[ntt] = (uint8_t)sm;
      int em = 0;
      for (int i = 0; i < 6; ++i) {
        int a = q[EDGES[i][0]], b = q[EDGES[i][1]];
        if (a != GHOST && b != GHOST && seg_keys.count(k2(a, b))) em |= 1 << i;
      }
      seg_mask[ntt] = (uint8_t)em;
      star_ratio(ntt);
    }
    vert_tet[vid] = nt0;
    return vid;
  }

  // _kernels.py:742-804 (float path) with the exact fallback of mesh.py:770-771
  void star_ratio(int t) {
    const int* q = &tv[4 * (size_t)t];
    if (q[3] == GHOST) { ratio[t] = -1.0; return; }
    const double *A = pt(q[0]), *Bp = pt(q[1]), *C = pt(q[2]), *D = pt(q[3]);
    double ax = A[0], ay = A[1], az = A[2];
    double ux = Bp[0] - ax, uy = Bp[1] - ay, uz = Bp[2] - az;
    double vx = C[0] - ax, vy = C[1] - ay, vz = C[2] - az;
    double wx = D[0] - ax, wy = D[1] - ay, wz = D[2] - az;
    double vwx = vy * wz - vz * wy, vwy = vz * wx - vx * wz, vwz = vx * wy - vy * wx;
    double denom = 2.0 * (ux * vwx + uy * vwy + uz * vwz);
    if (denom == 0.0 || !std::isfinite(denom)) { compute_ratio(t); return; }
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
    auto sq = [](const double* x, const double* y) {
      double e0 = x[0] - y[0], e1 = x[1] - y[1], e2 = x[2] - y[2];
      return e0 * e0 + e1 * e1 + e2 * e2; };
    double d2 = sq(C, Bp); if (d2 < sh) sh = d2;
    d2 = sq(D, Bp); if (d2 < sh) sh = d2;
    d2 = sq(D, C); if (d2 < sh) sh = d2;
    ratio[t] = std::sqrt(r2 / sh);
  }

  // mesh.py:847-865
  void compact() {
    std::vector<int> remap(nt, -1);
    int n = 0;
    for (int t = 0; t < nt; ++t) if (alive[t] == 1) remap[t] = n++;
    for (int t = 0; t < nt; ++t) {
      int r = remap[t];
      if (r < 0) continue;
      for (int k = 0; k < 4; ++k) {
        tv[4 * (size_t)r + k] = tv[4 * (size_t)t + k];
        int64_t x = tn[4 * (size_t)t + k];
        tn[4 * (size_t)r + k] = (int64_t)remap[x >> 2] * 4 + (x & 3);
      }
      sub_mask[r] = sub_mask[t]; seg_mask[r] = seg_mask[t];
      ratio[r] = ratio[t]; skip_flag[r] = skip_flag[t];
    }
    for (int t = 0; t < n; ++t) alive[t] = 1;
    for (int t = n; t < nt; ++t) alive[t] = 0;
    nt = n;
    for (int v = 0; v < nv; ++v) vert_tet[v] = vert_tet[v] >= 0 ? remap[vert_tet[v]] : -1;
  }

  // mesh.py:869-943; order = numpy default_rng(seed).shuffle(range(n)) computed by the caller
  void init_delaunay(const double* pts, int n, const int* order) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], pts[3 * i + k]); hi[k] = std::max(hi[k], pts[3 * i + k]); }
    set_bbox(lo, hi);
    for (int i = 0; i < n; ++i) add_vertex(&pts[3 * i], 0);
    auto collinear = [&](int a, int b, int c) {
      for (int axis = 0; axis < 3; ++axis) {
        int i = axis == 0 ? 1 : 0, j = axis == 2 ? 1 : 2;
        double a2[2] = {pt(a)[i], pt(a)[j]}, b2[2] = {pt(b)[i], pt(b)[j]}, c2[2] = {pt(c)[i], pt(c)[j]};
        if (orient2d(a2, b2, c2) != 0) return false;
      }
      return true;
    };
    std::vector<int> first{order[0]};
    for (int k = 1; k < n; ++k) {
      int idx = order[k];
      std::vector<int> cand = first; cand.push_back(idx);
      bool ok = false;
      if (cand.size() == 2) {
        const double *a = pt(cand[0]), *b = pt(cand[1]);
        ok = !(a[0] == b[0] && a[1] == b[1] && a[2] == b[2]);
      } else if (cand.size() == 3) ok = !collinear(cand[0], cand[1], cand[2]);
      else ok = orient3d(pt(cand[0]), pt(cand[1]), pt(cand[2]), pt(cand[3])) != 0;
      if (ok) first.push_back(idx);
      if (first.size() == 4) break;
    }
    if (first.size() < 4) throw std::runtime_error("no four non-coplanar points");
    int a = first[0], b = first[1], c = first[2], d = first[3];
    if (orient3d(pt(a), pt(b), pt(c), pt(d)) < 0) std::swap(a, b);
    int t0 = new_tet(a, b, c, d);
    std::vector<int> ghosts;
    for (int i = 0; i < 4; ++i) {
      int f[3]; face_verts(t0, i, f);
      int g = new_tet(f[0], f[1], f[2], GHOST);
      ghosts.push_back(g);
      set_nb(t0, i, g, 3);
    }
    std::map<K3, std::pair<int, int>> fmap;
    for (int g : ghosts) for (int i = 0; i < 3; ++i) {
      K3 key = face_key(g, i);
      auto it = fmap.find(key);
      if (it != fmap.end()) { set_nb(g, i, it->second.first, it->second.second); fmap.erase(it); }
      else fmap[key] = {g, i};
    }
    compute_ratio(t0);
    int hint = t0;
    std::unordered_set<int> done(first.begin(), first.end());
    if (std::getenv("ORACLE_PARALLEL_INIT")) {
      std::vector<int> pend;
      for (int k = 0; k < n; ++k) if (!done.count(order[k])) pend.push_back(order[k]);
      std::vector<int> hints(pend.size(), t0);
      size_t off = 0;
      int inserted = 4;
      while (off < pend.size()) {
        size_t nwin = std::min(pend.size() - off, (size_t)std::max(256, 2 * inserted));
        std::vector<Region> regs(nwin);
        for (size_t k = 0; k < nwin; ++k) {
          const double* p = pt(pend[off + k]);
          double pc[3] = {p[0], p[1], p[2]};
          int h = hints[off + k];
          if (h < 0 || h >= nt || !alive[h]) h = t0;
          int s0 = walk(pc, h);
          hints[off + k] = s0;
          regs[k] = delaunay_region(pc, {s0}, nullptr);
        }
        // greedy by order over claims
        std::unordered_set<int64_t> claimed;
        std::vector<char> acc(nwin, 0);
        for (size_t k = 0; k < nwin; ++k) {
          std::vector<int64_t> ks;
          for (int t : regs[k].tets) ks.push_back(t);
          for (auto& bf : regs[k].bfaces) {
            int64_t a = 4 * (int64_t)bf.first + bf.second, b = tn[4 * (size_t)bf.first + bf.second];
            ks.push_back((int64_t)1 << 40 | std::min(a, b));
          }
          bool clash = false;
          for (auto x : ks) if (claimed.count(x)) { clash = true; break; }
          for (auto x : ks) claimed.insert(x);   // pending points block later ones either way
          acc[k] = !clash;
        }
        std::vector<int> np, nh;
        for (size_t k = 0; k < nwin; ++k) {
          if (acc[k]) {
            const double* p = pt(pend[off + k]);
            double pc[3] = {p[0], p[1], p[2]};
            insert_point(pc, regs[k], 0, nullptr, {}, {}, pend[off + k]);
            ++inserted;
          } else { np.push_back(pend[off + k]); nh.push_back(hints[off + k]); }
        }
        size_t newoff = off + nwin - np.size();
        for (size_t k = 0; k < np.size(); ++k) { pend[newoff + k] = np[k]; hints[newoff + k] = nh[k]; }
        off = newoff;
      }
      return;
    }
    for (int k = 0; k < n; ++k) {
      int idx = order[k];
      if (done.count(idx)) continue;
      const double* p = pt(idx);
      double pc[3] = {p[0], p[1], p[2]};
      int seed = walk(pc, hint);
      Region R = delaunay_region(pc, {seed}, nullptr);
      insert_point(pc, R, 0, nullptr, {}, {}, idx);
      hint = vert_tet[idx];
    }
  }

  int n_real_tets() const {
    int c = 0;
    for (int t = 0; t < nt; ++t) if (alive[t] == 1 && tv[4 * (size_t)t + 3] != GHOST) ++c;
    return c;
  }
};

}  // namespace orc
