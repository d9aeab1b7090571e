// TEST INFRASTRUCTURE ONLY -- CPU oracle (see oracle/README.md).
//
// Per-polygon planar Delaunay triangulations, restating
// /root/reference/pkg/src/tetrefine/facets.py:30-420 and the exact PLC
// helpers of plc.py (_proj_axis, _point_in_polygon_2d).
#pragma once
#include "oracle_mesh.hpp"

namespace orc {

static const int GHOST2 = -1;
inline uint64_t dkey(int a, int b) { return ((uint64_t)(uint32_t)(a + 1) << 32) | (uint32_t)(b + 1); }

// plc.py:73-85: dominant axis of the exact fan normal of a planar cycle
inline int proj_axis(const std::vector<std::array<double, 3>>& pts) {
  int n = (int)pts.size();
  std::vector<double> xs;
  for (auto& q : pts) { xs.push_back(q[0]); xs.push_back(q[1]); xs.push_back(q[2]); }
  std::vector<BigInt> v(xs.size());
  scaled_ints(xs.data(), (int)xs.size(), v.data());
  BigInt N[3];
  for (int i = 1; i < n - 1; ++i) {
    BigInt u[3], w[3];
    for (int k = 0; k < 3; ++k) { u[k] = v[3 * i + k] - v[k]; w[k] = v[3 * (i + 1) + k] - v[k]; }
    N[0] = N[0] + (u[1] * w[2] - u[2] * w[1]);
    N[1] = N[1] + (u[2] * w[0] - u[0] * w[2]);
    N[2] = N[2] + (u[0] * w[1] - u[1] * w[0]);
  }
  for (int k = 0; k < 3; ++k) if (N[k].sign < 0) N[k].sign = 1;
  int best = 0;
  for (int k = 1; k < 3; ++k) if (cmp(N[k], N[best]) > 0) best = k;
  return best;
}

// facets.py:322-335
inline int poly_area_sign(const std::vector<std::array<double, 2>>& p2) {
  int n = (int)p2.size();
  std::vector<double> xs;
  for (auto& q : p2) { xs.push_back(q[0]); xs.push_back(q[1]); }
  std::vector<BigInt> v(xs.size());
  scaled_ints(xs.data(), (int)xs.size(), v.data());
  BigInt tot;
  for (int k = 0; k < n; ++k) {
    int j = (k + 1) % n;
    tot = tot + (v[2 * k] * v[2 * j + 1] - v[2 * j] * v[2 * k + 1]);
  }
  return tot.sign;
}

// plc.py:159-179 with q = centroid of three float points (exact rational)
inline bool centroid_in_polygon(const std::vector<std::array<double, 2>>& poly, const double* t0,
                                const double* t1, const double* t2) {
  int n = (int)poly.size();
  std::vector<double> xs;
  for (auto& q : poly) { xs.push_back(q[0]); xs.push_back(q[1]); }
  xs.push_back(t0[0]); xs.push_back(t0[1]); xs.push_back(t1[0]); xs.push_back(t1[1]);
  xs.push_back(t2[0]); xs.push_back(t2[1]);
  std::vector<BigInt> v(xs.size());
  scaled_ints(xs.data(), (int)xs.size(), v.data());
  BigInt three(3);
  BigInt Qx = v[2 * n] + v[2 * n + 2] + v[2 * n + 4];   // 3*qx
  BigInt Qy = v[2 * n + 1] + v[2 * n + 3] + v[2 * n + 5];
  for (int i = 0; i < n; ++i) {
    int j = (i + 1) % n;
    BigInt ax = v[2 * i], ay = v[2 * i + 1], bx = v[2 * j], by = v[2 * j + 1];
    BigInt o = (bx - ax) * (Qy - ay * three) - (by - ay) * (Qx - ax * three);
    if (o.sign == 0) {
      if ((cmp(Qx, ax * three) == 0 && cmp(Qy, ay * three) == 0) ||
          (cmp(Qx, bx * three) == 0 && cmp(Qy, by * three) == 0)) return true;
      BigInt dot = (Qx - ax * three) * (bx - ax) + (Qy - ay * three) * (by - ay);
      BigInt lsq = ((bx - ax) * (bx - ax) + (by - ay) * (by - ay)) * three;
      if (dot.sign > 0 && cmp(dot, lsq) < 0) return true;
    }
  }
  bool inside = false;
  for (int i = 0; i < n; ++i) {
    int j = (i + 1) % n;
    BigInt ax = v[2 * i], ay = v[2 * i + 1], bx = v[2 * j], by = v[2 * j + 1];
    bool c1 = cmp(ay * three, Qy) > 0, c2 = cmp(by * three, Qy) > 0;
    if (c1 != c2) {
      BigInt D = by - ay;
      BigInt S = (ax * three - Qx) * D + (Qy - ay * three) * (bx - ax);
      if (S.sign * D.sign > 0) inside = !inside;
    }
  }
  return inside;
}

struct Tri2D {
  std::unordered_map<int, std::array<double, 2>> pos;
  std::vector<std::array<int, 3>> tris;
  std::vector<uint8_t> tri_alive;
  int n_alive = 0;
  std::unordered_map<uint64_t, int> half;
  int last = -1;

  const double* P(int v) const { return pos.at(v).data(); }
  int add_tri(int a, int b, int c) {
    int tid = (int)tris.size();
    tris.push_back({a, b, c});
    tri_alive.push_back(1);
    ++n_alive;
    half[dkey(a, b)] = tid; half[dkey(b, c)] = tid; half[dkey(c, a)] = tid;
    return tid;
  }
  void remove_tri(int tid) {
    auto t = tris[tid];
    tri_alive[tid] = 0;
    --n_alive;
    int e[3][2] = {{t[0], t[1]}, {t[1], t[2]}, {t[2], t[0]}};
    for (auto& x : e) {
      auto it = half.find(dkey(x[0], x[1]));
      if (it != half.end() && it->second == tid) half.erase(it);
    }
  }
  int half_get(int a, int b) const {
    auto it = half.find(dkey(a, b));
    return it == half.end() ? -1 : it->second;
  }
  bool alive_tid(int tid) const { return tid >= 0 && tid < (int)tris.size() && tri_alive[tid]; }

  void bootstrap(const std::vector<int>& vids, const std::vector<std::array<double, 2>>& coords) {
    std::vector<int> pending, base;
    for (size_t k = 0; k < vids.size(); ++k) {
      int vid = vids[k];
      pos[vid] = coords[k];
      if (base.size() < 3) {
        std::vector<int> cand = base; cand.push_back(vid);
        bool ok = true;
        if (cand.size() == 2) ok = !(P(cand[0])[0] == P(cand[1])[0] && P(cand[0])[1] == P(cand[1])[1]);
        else if (cand.size() == 3) ok = orient2d(P(cand[0]), P(cand[1]), P(cand[2])) != 0;
        if (ok) base.push_back(vid); else pending.push_back(vid);
        if (base.size() == 3) {
          int a = base[0], b = base[1], c = base[2];
          if (orient2d(P(a), P(b), P(c)) < 0) std::swap(a, b);
          add_tri(a, b, c); add_tri(b, a, GHOST2); add_tri(c, b, GHOST2); add_tri(a, c, GHOST2);
          last = 0;
        }
      } else pending.push_back(vid);
    }
    if (base.size() < 3) throw DegenerateTri("all facet vertices collinear");
    for (int vid : pending) { auto q = pos[vid]; insert(vid, q, {}); }
  }

  // facets.py:92-105
  bool in_tri_region(int tid, const double* p) const {
    auto t = tris[tid];
    if (t[2] == GHOST2) {
      const double *pa = P(t[0]), *pb = P(t[1]);
      int s = orient2d(pa, pb, p);
      if (s != 0) return s > 0;
      double xs[6] = {p[0], p[1], pa[0], pa[1], pb[0], pb[1]};
      BigInt v[6];
      scaled_ints(xs, 6, v);
      BigInt d0 = (v[0] - v[2]) * (v[4] - v[2]) + (v[1] - v[3]) * (v[5] - v[3]);
      BigInt dl = (v[4] - v[2]) * (v[4] - v[2]) + (v[5] - v[3]) * (v[5] - v[3]);
      return d0.sign > 0 && cmp(d0, dl) < 0;
    }
    return incircle2d(P(t[0]), P(t[1]), P(t[2]), p) > 0;
  }
  int first_alive() const { for (size_t i = 0; i < tris.size(); ++i) if (tri_alive[i]) return (int)i; return -1; }

  // facets.py:107-129
  int find_seed(const double* p) const {
    int tid = alive_tid(last) ? last : first_alive();
    for (int s = 0; s < 4 * n_alive + 16; ++s) {
      auto t = tris[tid];
      if (t[0] == GHOST2 || t[1] == GHOST2 || t[2] == GHOST2) break;
      bool moved = false;
      int e[3][2] = {{t[0], t[1]}, {t[1], t[2]}, {t[2], t[0]}};
      for (auto& x : e) {
        if (orient2d(P(x[0]), P(x[1]), p) < 0) { tid = half_get(x[1], x[0]); moved = true; break; }
      }
      if (!moved) break;
    }
    if (in_tri_region(tid, p)) return tid;
    for (size_t i = 0; i < tris.size(); ++i) if (tri_alive[i] && in_tri_region((int)i, p)) return (int)i;
    throw CNSS("2D point in no triangle's region");
  }

  std::set<int> cavity(const double* p) const {
    int seed = find_seed(p);
    std::set<int> cav{seed};
    std::vector<int> stack{seed};
    while (!stack.empty()) {
      int tid = stack.back(); stack.pop_back();
      auto t = tris[tid];
      int e[3][2] = {{t[1], t[0]}, {t[2], t[1]}, {t[0], t[2]}};
      for (auto& x : e) {
        int nb = half_get(x[0], x[1]);
        if (nb >= 0 && !cav.count(nb) && in_tri_region(nb, p)) { cav.insert(nb); stack.push_back(nb); }
      }
    }
    return cav;
  }

  void expand_star(std::set<int>& cav, const double* p) const {
    bool changed = true;
    while (changed) {
      changed = false;
      std::vector<int> snap(cav.begin(), cav.end());
      for (int tid : snap) {
        auto t = tris[tid];
        int e[3][2] = {{t[0], t[1]}, {t[1], t[2]}, {t[2], t[0]}};
        for (auto& x : e) {
          int nb = half_get(x[1], x[0]);
          if (nb < 0 || cav.count(nb)) continue;
          if (x[0] == GHOST2 || x[1] == GHOST2) continue;
          if (orient2d(P(x[0]), P(x[1]), p) <= 0) { cav.insert(nb); changed = true; }
        }
      }
      if ((int)cav.size() == n_alive) throw CNSS("2D cavity expansion consumed the whole triangulation");
    }
  }

  std::set<int> component(const std::set<int>& cav, int seed) const {
    std::set<int> comp{seed};
    std::vector<int> stack{seed};
    while (!stack.empty()) {
      int tid = stack.back(); stack.pop_back();
      auto t = tris[tid];
      int e[3][2] = {{t[1], t[0]}, {t[2], t[1]}, {t[0], t[2]}};
      for (auto& x : e) {
        int nb = half_get(x[0], x[1]);
        if (nb >= 0 && cav.count(nb) && !comp.count(nb)) { comp.insert(nb); stack.push_back(nb); }
      }
    }
    return comp;
  }

  // facets.py:185-236 ; returns removed/added triangles (vertex tuples)
  void insert(int vid, std::array<double, 2> p2, const std::vector<int>& forced,
              std::vector<std::array<int, 3>>* removed = nullptr, std::vector<std::array<int, 3>>* added = nullptr) {
    pos[vid] = p2;
    const double* p = pos[vid].data();
    std::set<int> cav;
    if (!forced.empty()) {
      cav.insert(forced.begin(), forced.end());
      int seed = -1;
      try {
        std::set<int> own = cavity(p);
        seed = *own.begin();
        cav.insert(own.begin(), own.end());
      } catch (CNSS&) {}
      expand_star(cav, p);
      cav = component(cav, seed >= 0 ? seed : *cav.begin());
    } else {
      cav = cavity(p);
    }
    std::vector<std::array<int, 2>> bedges;
    for (int tid : cav) {
      auto t = tris[tid];
      if (removed) removed->push_back(t);
      int e[3][2] = {{t[0], t[1]}, {t[1], t[2]}, {t[2], t[0]}};
      for (auto& x : e) {
        int m = half_get(x[1], x[0]);
        if (m < 0 || !cav.count(m)) bedges.push_back({x[0], x[1]});
      }
    }
    for (int tid : cav) remove_tri(tid);
    for (auto& e : bedges) {
      int u = e[0], v = e[1], tid;
      if (u == GHOST2 || v == GHOST2) {
        if (u == GHOST2) { tid = add_tri(v, vid, GHOST2); if (added) added->push_back({v, vid, GHOST2}); }
        else { tid = add_tri(vid, u, GHOST2); if (added) added->push_back({vid, u, GHOST2}); }
      } else {
        tid = add_tri(u, v, vid);
        if (added) added->push_back({u, v, vid});
      }
      last = tid;
    }
  }
};

struct Facet {
  int pid;
  std::vector<int> corner_ids;
  int axis, keep[2];
  std::vector<std::array<double, 2>> poly2d;
  Tri2D tri;
  std::unordered_map<K3, bool, K3H> inside_cache;

  std::array<double, 2> project(const double* p3) const { return {p3[keep[0]], p3[keep[1]]}; }

  void init(int pid_, const std::vector<int>& ids, const std::vector<std::array<double, 3>>& pts) {
    pid = pid_;
    corner_ids = ids;
    axis = proj_axis(pts);
    int i = axis == 0 ? 1 : 0, j = axis == 2 ? 1 : 2;
    std::vector<std::array<double, 2>> p2;
    for (auto& q : pts) p2.push_back({q[i], q[j]});
    if (poly_area_sign(p2) < 0) std::swap(i, j);
    keep[0] = i; keep[1] = j;
    poly2d.clear();
    for (auto& q : pts) poly2d.push_back({q[i], q[j]});
    std::vector<std::array<double, 2>> coords;
    for (auto& q : pts) coords.push_back(project(q.data()));
    tri.bootstrap(corner_ids, coords);
  }

  bool tri_inside(const std::array<int, 3>& t) {
    if (t[0] == GHOST2 || t[1] == GHOST2 || t[2] == GHOST2) return false;
    K3 key = sort3(t[0], t[1], t[2]);
    auto it = inside_cache.find(key);
    if (it != inside_cache.end()) return it->second;
    bool hit = centroid_in_polygon(poly2d, tri.P(t[0]), tri.P(t[1]), tri.P(t[2]));
    inside_cache[key] = hit;
    return hit;
  }

  std::set<K3> subface_keys() {
    std::set<K3> out;
    for (size_t i = 0; i < tri.tris.size(); ++i)
      if (tri.tri_alive[i] && tri_inside(tri.tris[i])) out.insert(sort3(tri.tris[i][0], tri.tris[i][1], tri.tris[i][2]));
    return out;
  }

  // facets.py:297-319
  void insert(int vid, const double* p3, const std::vector<K3>& crossed, const uint64_t* split_edge,
              std::set<K3>& rem, std::set<K3>& add) {
    std::vector<int> forced;
    if (!crossed.empty()) {
      std::unordered_map<K3, int, K3H> kmap;
      for (size_t i = 0; i < tri.tris.size(); ++i) {
        if (!tri.tri_alive[i]) continue;
        auto& t = tri.tris[i];
        if (t[0] == GHOST2 || t[1] == GHOST2 || t[2] == GHOST2) continue;
        kmap[sort3(t[0], t[1], t[2])] = (int)i;
      }
      std::vector<K3> cs = crossed;
      std::sort(cs.begin(), cs.end());
      for (auto& k : cs) { auto it = kmap.find(k); if (it != kmap.end()) forced.push_back(it->second); }
    }
    if (split_edge) {
      int u = k2u(*split_edge), v = k2v(*split_edge);
      int t1 = tri.half_get(u, v); if (t1 >= 0) forced.push_back(t1);
      int t2 = tri.half_get(v, u); if (t2 >= 0) forced.push_back(t2);
    }
    std::vector<std::array<int, 3>> removed, added;
    tri.insert(vid, project(p3), forced, &removed, &added);
    for (auto& t : removed) if (tri_inside(t)) rem.insert(sort3(t[0], t[1], t[2]));
    for (auto& t : added) if (tri_inside(t)) add.insert(sort3(t[0], t[1], t[2]));
  }
};

struct FacetComplex {
  std::vector<Facet> facets;
  std::vector<std::vector<int>> segment_polygons;          // sid -> pids
  std::vector<std::set<K3>> keys_by_pid;
  std::unordered_map<int, std::set<int>> vert_sids;

  void init(const std::vector<double>& pts, const std::vector<std::array<int, 2>>& segs,
            const std::vector<std::vector<int>>& polys) {
    std::unordered_map<uint64_t, int> seg_index;
    for (size_t sid = 0; sid < segs.size(); ++sid) seg_index[k2(segs[sid][0], segs[sid][1])] = (int)sid;
    segment_polygons.assign(segs.size(), {});
    for (size_t sid = 0; sid < segs.size(); ++sid) {
      vert_sids[segs[sid][0]].insert((int)sid);
      vert_sids[segs[sid][1]].insert((int)sid);
    }
    facets.resize(polys.size());
    keys_by_pid.resize(polys.size());
    for (size_t pid = 0; pid < polys.size(); ++pid) {
      std::vector<std::array<double, 3>> cp;
      for (int v : polys[pid]) cp.push_back({pts[3 * v], pts[3 * v + 1], pts[3 * v + 2]});
      facets[pid].init((int)pid, polys[pid], cp);
      keys_by_pid[pid] = facets[pid].subface_keys();
      int n = (int)polys[pid].size();
      for (int k = 0; k < n; ++k) {
        int a = polys[pid][k], b = polys[pid][(k + 1) % n];
        segment_polygons[seg_index.at(k2(a, b))].push_back((int)pid);
      }
    }
  }

  bool collinear_sliver(const K3& key) {
    std::set<int> sids;
    bool first = true;
    for (int v : {key.a, key.b, key.c}) {
      auto it = vert_sids.find(v);
      if (it == vert_sids.end() || it->second.empty()) return false;
      if (first) { sids = it->second; first = false; }
      else {
        std::set<int> x;
        for (int s : sids) if (it->second.count(s)) x.insert(s);
        sids.swap(x);
      }
      if (sids.empty()) return false;
    }
    return true;
  }

  void apply(int pid, int vid, const double* p3, const std::vector<K3>& crossed, const uint64_t* split_edge,
             std::set<K3>& rem, std::set<K3>& add) {
    std::set<K3> r, a;
    facets[pid].insert(vid, p3, crossed, split_edge, r, a);
    for (auto& k : r) if (keys_by_pid[pid].count(k)) rem.insert(k);
    for (auto& k : a) if (!collinear_sliver(k)) add.insert(k);
    for (auto& k : rem) keys_by_pid[pid].erase(k);
    for (auto& k : add) keys_by_pid[pid].insert(k);
  }

  // facets.py:396-416
  void split_segment(int sid, uint64_t edge, int vid, const double* p3,
                     const std::map<int, std::vector<K3>>& crossed_by_pid,
                     std::vector<K3>& removed, std::vector<std::pair<K3, int>>& added) {
    vert_sids[vid].insert(sid);
    for (int pid : segment_polygons[sid]) {
      auto it = crossed_by_pid.find(pid);
      std::vector<K3> crossed = it == crossed_by_pid.end() ? std::vector<K3>() : it->second;
      std::set<K3> rem, add;
      apply(pid, vid, p3, crossed, &edge, rem, add);
      for (auto& k : rem) removed.push_back(k);
      for (auto& k : add) added.push_back({k, pid});
    }
    std::vector<K3> r2; std::set<K3> s1;
    for (auto& k : removed) if (!s1.count(k)) { s1.insert(k); r2.push_back(k); }
    removed.swap(r2);
    std::vector<std::pair<K3, int>> a2; std::set<K3> s2;
    for (auto& ka : added) if (!s2.count(ka.first)) { s2.insert(ka.first); a2.push_back(ka); }
    added.swap(a2);
  }

  void split_facet(int pid, int vid, const double* p3, const std::vector<K3>& crossed,
                   std::vector<K3>& removed, std::vector<std::pair<K3, int>>& added) {
    std::set<K3> rem, add;
    apply(pid, vid, p3, crossed, nullptr, rem, add);
    for (auto& k : rem) removed.push_back(k);
    for (auto& k : add) added.push_back({k, pid});
  }
};

}  // namespace orc
