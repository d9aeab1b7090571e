// gq_fallback.cuh -- sequential fallback for failed candidates (refine.py:748-799).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

// ---------------------------------------------------------------------------
// sequential fallback for failed candidates (refine.py:748-799): one thread,
// in pool order, on the updated mesh.  Uses the big scratch / slab 0.
struct FallbackIO { const int* list; int n; int round_no; unsigned long long seed; int with_facets; double lmin2; int* inserted;
                   int window;   // candidates evaluated per wave (waves)
};

__device__ inline void mark_enc_face_key(const Dev& D, int a, int b, int c) {
  sort3(a, b, c);
  int r = face_lookup(D, a, b, c);
  if (r >= 0 && !(D.sf_fl[r] & RF_SKIP)) D.sf_fl[r] |= RF_ENC;
}
__device__ __noinline__ void skip_cand(const Dev& D, const Cand& C, int c, int reason, int round_no, const SkipLog& L,
                                       int order) {
  int kind = C.kind[c], tgt = C.tgt[c];
  if (kind == K_TET) {
    if (tgt >= 0 && tgt < D.ctr->nt && D.alive[tgt]) {
      D.skip[tgt] = 1;
      int cv[4]; tet_canon(D, tgt, cv);
      log_skip(D, L, round_no, K_TET, reason, cv, 4, order);
    }
  } else if (kind == K_SEG) {
    D.sg_fl[tgt] = (D.sg_fl[tgt] | RF_SKIP) & ~RF_ENC;
    int2 e = D.sg_uv[tgt]; int v[2] = {e.x, e.y};
    log_skip(D, L, round_no, K_SEG, reason, v, 2, order);
  } else {
    D.sf_fl[tgt] = (D.sf_fl[tgt] | RF_SKIP) & ~RF_ENC;
    int4 f = D.sf_v[tgt]; int v[3] = {f.x, f.y, f.z};
    log_skip(D, L, round_no, K_FACE, reason, v, 3, order);
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
    // polygons of the split element: every polygon of the segment (any number), or the subface's
    int o0 = 0, np = 1, fpid = -1;
    if (C.kind[c] == K_SEG) {
      int sid = D.sg_sid[C.tgt[c]];
      o0 = D.segpoly_off[sid]; np = D.segpoly_off[sid + 1] - o0;
    } else fpid = D.sf_v[C.tgt[c]].w;
    if (item0 + np > T.icap) { raise_err(GQ_ERR_CAP); np = T.icap - item0; }
    for (int k = 0; k < np; ++k) {
      int w = item0 + k;
      int pid = fpid >= 0 ? fpid : D.segpoly[o0 + k];
      Tri2Ctx X; X.D = &D; X.pid = pid; X.vid = vid; X.follow3d = D.poly_obl[pid];
      proj2(D, pid, p, X.p);
      int forced[T2_FCAP + 1]; int nf;    // the crossed triangles, then (seeds) the target's own
      t2_forced(D, C, c, pid, forced, nf, T2_FCAP);
      const int* seeds = forced; int ns = nf;
      int ts = t2_seed_of(D, C, c, pid);
      if (ts >= 0) forced[ns++] = ts;
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
          if (!tri_in_polygon(D, pid, a, b, cc)) return;
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
  atomicAdd(&D.ctr->created, (unsigned long long)C.nbf[c]); atomicAdd(&D.ctr->deleted, (unsigned long long)C.ntet[c]);
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

// ---------------------------------------------------------------------------
// Sequential fallback (refine.py:748-806 _fallback, called in failed-list order
// at refine.py:897-902).  Each failed candidate is re-evaluated on the mesh left
// by the accepted insertions and by every earlier fallback.  Almost all of them
// fail again (C4 face rounds: ~1% insert), and a failing evaluation writes only
// flags, so the list runs in waves: k_fb_scan evaluates every remaining
// candidate in parallel on the current mesh, without side effects; k_fb_apply
// then applies, in list order, the outcomes of the candidates before the first
// one that inserts (or that exceeds the scan's arenas) -- they saw exactly the
// mesh the sequential loop would show them -- and runs that first candidate
// through the full sequential body.  The next wave starts after it.  Results,
// vertex ids and tet ids equal the one-candidate-at-a-time loop.
#define FB_NONE 0      // target gone
#define FB_TOOCLOSE 1  // skip, reason too_close
#define FB_HULL 2      // tet: a hull subface obstructs it (arg = face record, -1 none)
#define FB_SHORT 3     // tet: short boundary edge
#define FB_MEMB 4      // membrane (arg = 4t+i)
#define FB_CNSS 5      // skip, reason cavity_not_star_shaped
#define FB_BREAK 6     // inserts (or needs the sequential arenas): run the full body
#define FB_OVF 7       // the concurrent cavity overflowed every tier (> 64k tets): beyond the
                       // sequential arena (8192 tets) too, skipped without re-growing it

// evaluation of failed candidate k; commit=false: no writes except the
// candidate's own arrays (returns the outcome), commit=true: the sequential body
__device__ __noinline__ int fallback_eval(const Dev& D, const Cand& C, Scratch& S, const FallbackIO& F, T2Items& T,
                                          const SkipLog& L, int k, bool commit, int* arg) {
  CandCtx X; X.round_no = F.round_no; X.seed = F.seed; X.with_facets = F.with_facets;
  int c = F.list[k];
  int kind = C.kind[c], tgt = C.tgt[c];
  if (C.status[c] == CS_TOOCLOSE) { if (commit) skip_cand(D, C, c, 2, F.round_no, L, skip_order(2, k)); return FB_TOOCLOSE; }
  if (kind == K_TET && !(tgt >= 0 && tgt < D.ctr->nt && D.alive[tgt])) return FB_NONE;
  if (kind == K_SEG && !(D.sg_fl[tgt] & RF_LIVE)) return FB_NONE;
  if (kind == K_FACE && !(D.sf_fl[tgt] & RF_LIVE)) return FB_NONE;
  if (C.status[c] == CS_CNSS && C.memb[c] == MEMB_HUGE_OVF) {
    if (commit) { atomicAdd(&D.ctr->fail[5], 1u); skip_cand(D, C, c, 3, F.round_no, L, skip_order(2, k)); }
    return FB_OVF;
  }
  long long tc0 = clock64();
  if (!make_cand(D, C, c, X, S)) { if (commit) raise_err(GQ_ERR_DEGEN); return commit ? FB_NONE : FB_BREAK; }
  long long tc1 = clock64(), tc2 = tc1;
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
      if (commit) { if (!(D.sf_fl[hull] & RF_SKIP)) D.sf_fl[hull] |= RF_ENC; }
      *arg = hull;
      return FB_HULL;
    }
  }
  tc2 = clock64();
  C.bigi[c] = commit ? 0 : -1;     // sequential: big slab 0; scan: the candidate's own slab
  SlabView sv = slab(C, c);
  RegionOut O = region_view(C, c, sv, 0);
  int seeds[32];
  int ns = cand_seeds(D, C, c, seeds, S);
  atomicAdd(&D.ctr->region_calls, 1ull);
  long long tc3 = clock64();
  int st = ns == 0 ? RS_CNSS : region_compute(D, p, seeds, ns, allow_of(C, c), S, O);
  long long tc4 = clock64();
  if (!commit && tc4 - tc0 > 19650000ll) {   // diagnostics: where a slow evaluation spends its time
    atomicAdd(&D.ctr->vq[6], (unsigned long long)((tc1 - tc0) >> 10)); atomicAdd(&D.ctr->vq[7], (unsigned long long)((tc2 - tc1) >> 10));
    atomicAdd(&D.ctr->vq[8], (unsigned long long)((tc3 - tc2) >> 10)); atomicAdd(&D.ctr->vq[9], (unsigned long long)((tc4 - tc3) >> 10));
    atomicAdd(&D.ctr->vq[10], 1ull);
  }
  store_region(C, c, O);
  if (st == RS_OK) {
    if (O.mind <= D.too_close_sq) { if (commit) skip_cand(D, C, c, 2, F.round_no, L, skip_order(2, k)); return FB_TOOCLOSE; }
    if (kind == K_TET && O.mind < F.lmin2) {
      if (commit) {
        D.skip[tgt] = 1;
        int cv[4]; tet_canon(D, tgt, cv);
        log_skip(D, L, F.round_no, K_TET, 1, cv, 4, skip_order(2, k));
      }
      return FB_SHORT;
    }
    if (!commit) return FB_BREAK;
    if (D.ctr->nv >= D.vcap) { raise_err(GQ_ERR_CAP); return FB_BREAK; }
    insert_one(D, C, c, S, T, 0);
    atomicAdd(F.inserted, 1);
    return FB_BREAK;
  } else if (st == RS_MEMBRANE) {
    if (commit) {
      int t = O.memb >> 2, i = O.memb & 3;
      int f[3]; face_verts(D.tv[t], i, f);
      mark_enc_face_key(D, f[0], f[1], f[2]);
      if (kind == K_SEG) D.sg_fl[tgt] |= RF_BLOCK;
      else if (kind == K_FACE) D.sf_fl[tgt] |= RF_BLOCK;
    }
    *arg = O.memb;
    return FB_MEMB;
  }
  if (st == RS_OVERFLOW && !commit) return FB_BREAK;   // the sequential arenas may hold it
  if (commit) {
    if (st == RS_OVERFLOW) atomicAdd(&D.ctr->fail[5], 1u);
    // not star-shaped, or a cavity beyond the sequential path's arena
    // (8192 tets): skipped like the reference's CavityNotStarShaped
    skip_cand(D, C, c, 3, F.round_no, L, skip_order(2, k));
  }
  return FB_CNSS;
}

// the sequential loop (one thread), kept for GQ_FALLBACK_SERIAL comparisons
__global__ void k_fallback(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Scr SCB, FallbackIO F, T2Items T, SkipLog L) {
  if (blockIdx.x || threadIdx.x) return;
  Scratch S = scratch_for(SCB, 0);
  int arg = 0;
  for (int k = 0; k < F.n; ++k) fallback_eval(D, C, S, F, T, L, k, true, &arg);
}

// wave step 1: outcomes of the window [start, start + F.window) on the current
// mesh, and the first one that breaks the wave (atomicMin into *first, preset
// to the window's end).  The window keeps a slow evaluation late in the list
// (a subsegment whose midpoint walk crosses the box gap: ~25 ms on one thread)
// from being repeated in every wave.
__global__ void k_fb_scan(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const __grid_constant__ Scr SC,
                          FallbackIO F, T2Items T, SkipLog L, const int* startp, int* out, int* first) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  Scratch S = scratch_for(SC, tid);
  const int start = *startp, wend = min(F.n, start + F.window);
  for (int k = start + tid; k < wend; k += gridDim.x * blockDim.x) {
    int arg = -1;
    S.cancel = first; S.me = k;
    if (*(const volatile int*)first < k) { out[2 * k] = FB_CNSS; out[2 * k + 1] = -1; continue; }   // unused
    long long t0 = clock64();
    int o = fallback_eval(D, C, S, F, T, L, k, false, &arg);
    unsigned long long dt = (unsigned long long)(clock64() - t0);
    atomicMax(&D.ctr->fb_slow, (dt << 8) | (unsigned long long)(o << 4) | (unsigned long long)C.kind[F.list[k]]);
    out[2 * k] = o; out[2 * k + 1] = arg;
    if (o == FB_BREAK) atomicMin(first, k);
  }
}

// wave step 2 (one thread): apply the outcomes of [start, first) in list order,
// then the full sequential body for candidate first when it broke the window;
// the next wave starts after it (or at the window's end)
__global__ void k_fb_apply(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Scr SCB, FallbackIO F, T2Items T,
                           SkipLog L, int* startp, const int* out, int* first) {
  if (blockIdx.x || threadIdx.x) return;
  const int start = *startp, f = *first, wend = min(F.n, start + F.window);
  for (int k = start; k < f; ++k) {
    int c = F.list[k];
    int kind = C.kind[c], tgt = C.tgt[c];
    int o = out[2 * k], arg = out[2 * k + 1];
    if (o == FB_OVF) atomicAdd(&D.ctr->fail[5], 1u);
    if (o == FB_TOOCLOSE || o == FB_CNSS || o == FB_OVF) {
      skip_cand(D, C, c, o == FB_TOOCLOSE ? 2 : 3, F.round_no, L, skip_order(2, k));
    } else if (o == FB_HULL) {
      if (!(D.sf_fl[arg] & RF_SKIP)) D.sf_fl[arg] |= RF_ENC;
    } else if (o == FB_SHORT) {
      D.skip[tgt] = 1;
      int cv[4]; tet_canon(D, tgt, cv);
      log_skip(D, L, F.round_no, K_TET, 1, cv, 4, skip_order(2, k));
    } else if (o == FB_MEMB) {
      int t = arg >> 2, i = arg & 3;
      int fv[3]; face_verts(D.tv[t], i, fv);
      mark_enc_face_key(D, fv[0], fv[1], fv[2]);
      if (kind == K_SEG) D.sg_fl[tgt] |= RF_BLOCK;
      else if (kind == K_FACE) D.sf_fl[tgt] |= RF_BLOCK;
    }
  }
  int next = wend;
  if (f < wend) {
    Scratch S = scratch_for(SCB, 0);
    int arg = 0;
    fallback_eval(D, C, S, F, T, L, f, true, &arg);
    next = f + 1;
  }
  *startp = next;
  *first = min(F.n, next + F.window);
}

// accepted tets whose region has a too-short boundary edge (refine.py:891-894)
__global__ void k_accept_flags(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* acc, int nacc, int* insflag, SkipLog L, int round_no, double lmin2) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nacc; k += gridDim.x * blockDim.x) {
    int c = acc[k];
    if (C.kind[c] == K_TET && C.mind[c] < lmin2) {
      insflag[k] = 0;
      int t = C.tgt[c];
      if (t >= 0 && D.alive[t]) {
        D.skip[t] = 1;
        int cv[4]; tet_canon(D, t, cv);
        log_skip(D, L, round_no, K_TET, 1, cv, 4, skip_order(1, k));
      }
    } else insflag[k] = 1;
  }
}
__global__ void k_assign_ids(const __grid_constant__ Cand C, const int* ins, int n, const int* nbfscan, int nv0, int nt0) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int c = ins[k];
    C.vid[c] = nv0 + k;
    C.nt0[c] = nt0 + nbfscan[k];
  }
}
__global__ void k_gather_nbf(const __grid_constant__ Cand C, const int* ins, int n, int* out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = C.nbf[ins[k]];
}
__global__ void k_rank_scatter(const __grid_constant__ Cand C, const int* order, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) C.rank[order[k]] = k;
}

// compaction of dead tet slots (mesh.py:847-865), stable
__global__ void k_compact_flags(const __grid_constant__ Dev D, int* flags) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) flags[t] = D.alive[t] == 1;
}
__global__ void k_compact_move(const __grid_constant__ Dev D, const int* remap, int nt, TetRow tv2, TetRow tn2, uint8_t* sub2, uint8_t* seg2,
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
__global__ void k_compact_vt(const __grid_constant__ Dev D, const int* remap, const int* flags, int nv) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int t = D.vert_tet[v];
    D.vert_tet[v] = t >= 0 ? (flags[t] ? remap[t] : -1) : -1;
  }
}

// quality (stats.py:35-99): bad count + dihedral histogram of real tets
// Dihedral angles within 1e-11 of a 5-degree bin edge depend on the last bit
// of acos (CUDA's vs the C library's numpy calls): such tets are listed for the
// host, which bins them with the reference's own numpy expression
// (stats.py:64-86), and left out of the device histogram.
__device__ inline bool bin_edge(double ang) {
  double x = ang / 5.0;
  return fabs(x - rint(x)) < 1e-11 * fmax(1.0, x);
}
__global__ void k_quality(const __grid_constant__ Dev D, double B, unsigned long long* bad, unsigned long long* hist, int* edge_list,
                          int edge_cap, int* n_edge) {
  // per-block counts in shared memory, one global add per bin per block
  __shared__ unsigned int s_cnt[37];   // [0] bad, [1 + b] histogram bin b
  for (int i = threadIdx.x; i < 37; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
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
    if (ratio > B) atomicAdd(&s_cnt[0], 1u);
    int bins[6];
    bool edge = false;
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
      else if (bin_edge(ang)) edge = true;
      bins[e] = bin;
    }
    if (edge) {
      int k = atomicAdd(n_edge, 1);
      if (k < edge_cap) { edge_list[k] = t; continue; }
    }
    for (int e = 0; e < 6; ++e) atomicAdd(&s_cnt[1 + bins[e]], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 37; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(i == 0 ? bad : hist + (i - 1), (unsigned long long)s_cnt[i]);
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


// ---------------------------------------------------------------------------
// Star validation of the accepted set, before anything is written.  The peel
// leaves every boundary face strictly visible from p, but a cavity whose
// boundary pinches along an edge (two wedges of tets meeting at it, one of
// them reflex) passes that test and cannot be starred; neither can a ghost
// cavity of a point rounded just outside a curved hull.  The reference meets
// such cavities only while starring (star_kernel's unmatched-face status,
// _kernels.py:696,720 -> CavityNotStarShaped, mesh.py:769-770): inside
// _fallback it skips the element (refine.py:785-799), on the main path the
// exception ends the refine.  Here an accepted candidate whose boundary faces
// do not pair up is skipped with reason cavity_not_star_shaped and nothing is
// inserted for it.  Same pairing as star_warp (gq_warp.cuh), no writes.
__device__ inline bool star_pairs_ok(const Dev& D, const int* bf, int nbf, const StarHash& X) {
  const int lane = threadIdx.x & 31;
  const int vid = -2;                       // the new vertex (no id yet); not GHOST, not a vertex id
  for (int i = lane; i < X.cap; i += 32) { X.key[i] = EMPTY_KEY; X.v0[i] = -1; X.v1[i] = -1; }
  if (lane == 0) *X.flag = 0;
  __syncwarp();
  for (int k = lane; k < nbf; k += 32) {
    int t = bf[k] >> 2, i = bf[k] & 3;
    int packed = tnk(D, t, i);
    int u = packed >> 2, j = packed & 3;
    int f[3]; face_verts(D.tv[u], j, f);
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
      int mine = 4 * k + m;
      if (atomicCAS(&X.v0[h], -1, mine) != -1 && atomicCAS(&X.v1[h], -1, mine) != -1) *X.flag = 1;
    }
    if (om < 0) *X.flag = 1;
  }
  __syncwarp();
  for (int k = lane; k < nbf && !*X.flag; k += 32) {
    int t = bf[k] >> 2, i = bf[k] & 3;
    int packed = tnk(D, t, i);
    int f[3]; face_verts(D.tv[packed >> 2], packed & 3, f);
    int4 q = (f[0] == GHOST || f[1] == GHOST || f[2] == GHOST) ? make_int4(0, 0, 0, GHOST) : make_int4(f[0], f[1], f[2], vid);
    if (q.w == GHOST) {
      int e0, e1;
      if (f[0] == GHOST) { e0 = f[1]; e1 = f[2]; }
      else if (f[1] == GHOST) { e0 = f[2]; e1 = f[0]; }
      else { e0 = f[0]; e1 = f[1]; }
      q = make_int4(e1, e0, vid, GHOST);
    }
    for (int m = 0; m < 4; ++m) {
      int g[3]; face_verts(q, m, g);
      if (g[0] != vid && g[1] != vid && g[2] != vid) continue;
      int h = star_slot(X, inner_key(g, vid), false);
      int mine = 4 * k + m;
      int other = h < 0 ? -1 : (X.v0[h] == mine ? X.v1[h] : X.v0[h]);
      if (other < 0) *X.flag = 1;
    }
  }
  __syncwarp();
  return *X.flag == 0;
}
__global__ void __launch_bounds__(32 * WS_WARPS) k_star_check(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* acc, int nacc, int* insflag,
                                                            const __grid_constant__ Scr SB, SkipLog L, int round_no) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StarShared& X = reinterpret_cast<StarShared*>(smem_raw)[wib];
  const int gw = blockIdx.x * WS_WARPS + wib, nw = gridDim.x * WS_WARPS;
  for (int k = gw; k < nacc; k += nw) {
    if (!insflag[k]) continue;
    int c = acc[k];
    SlabView v = slab(C, c);
    int nbf = C.nbf[c];
    bool ok;
    if (nbf <= WS_MAXF) ok = star_pairs_ok(D, v.bf, nbf, star_hash_shared(X));
    else if (C.bigi[c] >= HUGE_BASE) ok = star_pairs_ok(D, v.bf, nbf, huge_star_hash(C, c, &X.flag));
    else ok = star_pairs_ok(D, v.bf, nbf, big_star_hash(SB, gw, &X.flag));
    if (!ok && lane == 0) {
      atomicAdd(&D.ctr->fail[4], 1u);
      insflag[k] = 0;
      skip_cand(D, C, c, 3, round_no, L, skip_order(1, k));
    }
    __syncwarp();
  }
}
