// gq_init.cuh -- bulk Delaunay construction kernels, compaction, quality scan (mesh.py:847-943, stats.py:26-99).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

// ---------------------------------------------------------------------------
// bulk Delaunay construction (mesh.py:869-943) as priority rounds: every
// pending point in a prefix window of the insertion order computes its
// cavity; the filter accepts points whose claims avoid every lower-order
// pending point, which makes the result the sequential one.
__global__ void k_init_first(const __grid_constant__ Dev D, const int* order, int n, int* first_out) {
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
__global__ void k_init_region(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const __grid_constant__ Scr SC, const int* pend, const int* plist, int W, int* hint,
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
    atomicAdd(&D.ctr->region_calls, 1ull);
    int r = region_compute(D, p, seeds, 1, A, S, O, true);
    store_region(C, c, O);
    C.extra[c] = -1; C.kind[c] = K_TET; C.rank[c] = c; C.memb[c] = round;
    if (r == RS_OK) { C.status[c] = CS_OK; atomicAdd(&D.ctr->tested, (unsigned long long)(O.ntet + O.nbf)); }
    else if (r == RS_OVERFLOW) { C.status[c] = CS_OVF; C.memb[c] = -1; if (big) raise_err(GQ_ERR_CAP); }
    else { C.status[c] = CS_CNSS; raise_err(GQ_ERR_DEGEN); }
  }
}
// window filter: claims of every window point, strict lower-order rule
__global__ void k_init_claim(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, const int* plist, int nw) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    int c = plist[w];
    for_claims(D, C, W, c, [&](int k) { atomicMin(W.own + k, c); });
  }
}
__global__ void k_init_decide(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, const int* plist, int nw, int* acc) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    int c = plist[w];
    bool win = true;
    for_claims(D, C, W, c, [&](int k) { if (W.own[k] != c) win = false; });
    acc[w] = win ? 1 : 0;
  }
}
__global__ void k_init_unclaim(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, const int* plist, int nw) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    for_claims(D, C, W, plist[w], [&](int k) { W.own[k] = INT_MAX; });
}
// The window filter, tet-id assignment and cavity removal of one bulk round as
// one cooperative kernel: a warp per window point walks its claims
// lane-parallel; block 0 scans acceptance and boundary-face counts between the
// barriers; totals go to tot[0] (accepted) and tot[1] (new tets).
template <bool ONE>
__global__ void __launch_bounds__(256) k_init_filter_coop(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, const int* plist, int nw_in, int nt,
                                                          int* acc, int* accscan, int* nbfscan, int* tot, int* succ) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  const unsigned FULL = 0xffffffffu;
  // the window ends before the first point whose cavity overflowed the warp
  // kernel (it is computed by the block kernel next round): tot[3] = window,
  // tot[2] = overflowed points in the window
  if (blockIdx.x == 0 && threadIdx.x == 0) { tot[2] = 0; tot[3] = nw_in; }
  gsync<ONE>();
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw_in; w += gridDim.x * blockDim.x)
    if (C.status[plist[w]] == CS_OVF) { atomicMin(tot + 3, w); atomicAdd(tot + 2, 1); }
  gsync<ONE>();
  const int nw = *(volatile int*)(tot + 3);
  for (int w = nw + blockIdx.x * blockDim.x + threadIdx.x; w < nw_in; w += gridDim.x * blockDim.x) acc[w] = 0;
  for (int w = gw; w < nw; w += nwarp) {                    // claim: lowest order wins
    const int c = plist[w];
    warp_claims(D, C, W, c, lane, [&](int k) { atomicMin(W.own + k, c); });
  }
  gsync<ONE>();
  for (int w = gw; w < nw; w += nwarp) {                    // decide
    const int c = plist[w];
    bool win = true;
    warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] != c) win = false; });
    win = __all_sync(FULL, win);
    if (lane == 0) acc[w] = win;
  }
  gsync<ONE>();
  for (int w = gw; w < nw; w += nwarp)                      // release
    warp_claims(D, C, W, plist[w], lane, [&](int k) { W.own[k] = INT_MAX; });
  if (blockIdx.x == 0) {                                    // scans in insertion order
    typedef cub::BlockScan<int, 256> BS;
    __shared__ typename BS::TempStorage ts;
    __shared__ int carry[2];
    if (threadIdx.x == 0) carry[0] = carry[1] = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nw_in; b0 += 256) {   // the whole window: acc is 0 past the cut
      const int w = b0 + threadIdx.x;
      const int a = w < nw_in ? acc[w] : 0;
      const int f = a ? C.nbf[plist[w]] : 0;
      int sa, sf, ta, tf;
      BS(ts).ExclusiveSum(a, sa, ta);
      __syncthreads();
      BS(ts).ExclusiveSum(f, sf, tf);
      if (w < nw_in) { accscan[w] = carry[0] + sa; nbfscan[w] = carry[1] + sf; }
      __syncthreads();
      if (threadIdx.x == 0) { carry[0] += ta; carry[1] += tf; }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      tot[0] = carry[0]; tot[1] = carry[1];
      if (nt + carry[1] > D.tcap) raise_err(GQ_ERR_CAP);
    }
  }
  gsync<ONE>();
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
__global__ void k_init_nbf(const __grid_constant__ Cand C, const int* plist, const int* acc, int nw, int* nbfv) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    nbfv[w] = acc[w] ? C.nbf[plist[w]] : 0;
}
__global__ void k_init_kill(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* plist, const int* acc, const int* scan, int nw, int nt,
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
__global__ void k_init_stars(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* pend, const int* plist, const int* acc, int nw,
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
__global__ void k_count_ovf(const const __grid_constant__ Cand C, const int* plist, int W, int* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x)
    if (C.status[plist[w]] == CS_OVF) atomicAdd(out, 1);
    else if (C.status[plist[w]] == CS_OK) atomicMax(out + 1, C.ntet[plist[w]]);
}
__global__ void k_gather_status(const const __grid_constant__ Cand C, const int* plist, int W, int* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) out[w] = C.status[plist[w]];
}
__global__ void k_release_big(const __grid_constant__ Cand C, const int* list, int n) {
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
__global__ void k_facets_init(const __grid_constant__ Dev D, const int* poff, const int* pidx, int f, const __grid_constant__ Scr SC, int* t2base) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  for (int pid = tid; pid < f; pid += gridDim.x * blockDim.x) {
    int o0 = poff[pid], o1 = poff[pid + 1];
    Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = -2; X.follow3d = 0;
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
__global__ void k_facets_records(const __grid_constant__ Dev D, int nt2) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt2; t += gridDim.x * blockDim.x) {
    if (!D.t2alive[t]) continue;
    int4 q = D.t2v[t];
    if (q.z == GHOST) continue;
    if (!tri_in_polygon(D, q.w, q.x, q.y, q.z)) continue;   // facets.py:278-291 (non-convex polygons)
    new_face_record(D, q.x, q.y, q.z, q.w, RF_LIVE);
  }
}
__global__ void k_segs_init(const __grid_constant__ Dev D, const int* seg, int m) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    int u = seg[2 * s], v = seg[2 * s + 1];
    if (u > v) { int t = u; u = v; v = t; }
    D.sg_uv[s] = make_int2(u, v); D.sg_sid[s] = s; D.sg_fl[s] = RF_LIVE;
    D.sid_uv[s] = make_int2(u, v);
    ht_put(D.sg_hk, D.sg_hv, D.sg_hmask, key2(u, v), s);
  }
}
__global__ void k_refresh_all(const __grid_constant__ Dev D) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x)
    if (D.alive[t]) refresh_masks(D, t);
}

