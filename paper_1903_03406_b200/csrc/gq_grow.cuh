// gq_grow.cuh -- capacity management of the device mesh between and inside
// rounds.  The reference grows its numpy arrays by doubling whenever an
// insertion needs room (mesh.py:115-141); here every array is sized up front
// and grown the same way when a round is about to outgrow it:
//   * vertices and tet slots grow by copying (ids unchanged, so tet ids keep
//     matching the reference's; compaction stays on the reference's trigger);
//   * subsegment / subface records and facet 2D triangles are append-only
//     with dead entries left behind, so they are first compacted (stable,
//     hash tables rebuilt -- their ids never leave a round) and grown only if
//     the live ones still fill a quarter of the capacity.
// Part of the single translation unit gq_main.cu (included from gq_host.cuh).
#pragma once

__global__ void k_live_flags(const unsigned int* fl, int n, int* flags) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) flags[r] = (fl[r] & RF_LIVE) ? 1 : 0;
}
__global__ void k_move_seg_records(const __grid_constant__ Dev D, const int* flags, const int* scan, int n, int2* uv2, int* sid2, unsigned int* fl2) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (!flags[r]) continue;
    int q = scan[r];
    uv2[q] = D.sg_uv[r]; sid2[q] = D.sg_sid[r]; fl2[q] = D.sg_fl[r];
  }
}
__global__ void k_move_face_records(const __grid_constant__ Dev D, const int* flags, const int* scan, int n, int4* v2, unsigned int* fl2) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (!flags[r]) continue;
    int q = scan[r];
    v2[q] = D.sf_v[r]; fl2[q] = D.sf_fl[r];
  }
}
__global__ void k_rehash_segs(const __grid_constant__ Dev D, int n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int2 e = D.sg_uv[r];
    ht_put(D.sg_hk, D.sg_hv, D.sg_hmask, key2(e.x, e.y), r);
  }
}
__global__ void k_rehash_faces(const __grid_constant__ Dev D, int n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int4 f = D.sf_v[r];
    ht_put(D.sf_hk, D.sf_hv, D.sf_hmask, key3(f.x, f.y, f.z), r);
  }
}
__global__ void k_t2_live(const __grid_constant__ Dev D, int n, int* flags) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) flags[t] = D.t2alive[t] ? 1 : 0;
}
__global__ void k_t2_move(const __grid_constant__ Dev D, const int* flags, const int* scan, int n, int4* v2) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    if (flags[t]) v2[scan[t]] = D.t2v[t];
}
__global__ void k_t2_rehash(const __grid_constant__ Dev D, int n) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    int4 q = D.t2v[t];
    ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(q.x, q.y, q.w), t);
    ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(q.y, q.z, q.w), t);
    ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(q.z, q.x, q.w), t);
  }
}
__global__ void k_t2_last_remap(const __grid_constant__ Dev D, const int* flags, const int* scan) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < D.npoly; p += gridDim.x * blockDim.x) {
    int t = D.t2last[p];
    D.t2last[p] = (t >= 0 && flags[t]) ? scan[t] : -1;
  }
}

// new allocation of `cap` elements holding the first `used` of p (the rest
// memset to byte `fill` when fill >= 0); the old block goes back to the cache
template <class T>
static void regrow(gq_ctx* c, T*& p, size_t used, size_t cap, int fill = -1) {
  T* q = dmalloc<T>(cap);
  if (fill >= 0) CK(cudaMemsetAsync(q, fill, cap * sizeof(T), c->st));
  if (used) CK(cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, c->st));
  dfree(p);
  p = q;
}

// filter owner slots: [tets | faces (4*tcap) | subsegment records]; all INT_MAX between filters
static void realloc_owners(gq_ctx* c) {
  size_t n = 5 * (size_t)c->D.tcap + (size_t)c->D.sgcap;
  dfree(c->W.own);
  c->W.toff = 0; c->W.foff = c->D.tcap; c->W.soff = 5 * c->D.tcap;
  c->W.own = dmalloc<int>(n);
  CK(cudaMemsetAsync(c->W.own, 0x7f, n * 4, c->st));
}
static void realloc_grid_nodes(gq_ctx* c) {
  size_t cap = std::min<size_t>(((size_t)c->D.sgcap + c->D.sfcap) * 27, (size_t)1 << 30);
  if ((int)cap == c->G.node_cap) return;
  dfree(c->G.codes);
  c->G.node_cap = (int)cap;
  c->G.codes = dmalloc<int>(cap);
}

// room for nv_need vertices and nt_need tet slots
static void ensure_mesh_room(gq_ctx* c, long long nv_need, long long nt_need) {
  Dev& D = c->D;
  if (nv_need > D.vcap) {
    size_t cap = std::max<size_t>((size_t)nv_need + 65536, 2 * (size_t)D.vcap);
    if (cap > (size_t)INT_MAX / 4) throw std::runtime_error("vertex capacity beyond 32-bit ids");
    size_t nv = (size_t)c->hc.nv;
    regrow(c, D.P, 3 * nv, 3 * cap);
    regrow(c, D.vorigin, nv, cap);
    regrow(c, D.vert_tet, nv, cap, 0xff);
    regrow(c, D.vsid, nv, cap, 0xff);
    D.vcap = (int)cap;
    if (g_trace) std::fprintf(stderr, "[grow] vertices -> %zu\n", cap);
  }
  if (nt_need > D.tcap) {
    size_t cap = std::max<size_t>((size_t)nt_need + 65536, 2 * (size_t)D.tcap);
    if (5 * cap + (size_t)D.sgcap > (size_t)INT_MAX) throw std::runtime_error("tet capacity beyond 32-bit ids");
    size_t nt = (size_t)c->hc.nt;
    regrow(c, D.tv.p, 2 * nt, 2 * cap);
    D.tn.p = D.tv.p + 1;
    regrow(c, D.alive, nt, cap, 0);
    regrow(c, D.sub, nt, cap);
    regrow(c, D.seg, nt, cap);
    regrow(c, D.skip, nt, cap);
    regrow(c, D.ratio, nt, cap);
    D.tcap = (int)cap;
    // compaction double buffers are re-made at the new size on demand
    for (void* p : {(void*)c->tvn2, (void*)c->sub2, (void*)c->seg2, (void*)c->ratio2, (void*)c->skip2}) if (p) dfree(p);
    c->tvn2 = nullptr; c->sub2 = c->seg2 = c->skip2 = nullptr; c->ratio2 = nullptr;
    realloc_owners(c);
    if (g_trace) std::fprintf(stderr, "[grow] tets -> %zu\n", cap);
  }
}

static int scan_total(gq_ctx* c, const int* in, int* out, int n);

__global__ void k_rehash_live_segs(const __grid_constant__ Dev D, int n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    if (D.sg_fl[r] & RF_LIVE) { int2 e = D.sg_uv[r]; ht_put(D.sg_hk, D.sg_hv, D.sg_hmask, key2(e.x, e.y), r); }
}
__global__ void k_rehash_live_faces(const __grid_constant__ Dev D, int n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    if (D.sf_fl[r] & RF_LIVE) { int4 f = D.sf_v[r]; ht_put(D.sf_hk, D.sf_hv, D.sf_hmask, key3(f.x, f.y, f.z), r); }
}
__global__ void k_t2_rehash_live(const __grid_constant__ Dev D, int n) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (!D.t2alive[t]) continue;
    int4 q = D.t2v[t];
    ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(q.x, q.y, q.w), t);
    ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(q.y, q.z, q.w), t);
    ht_put(D.he_hk, D.he_hv, D.he_hmask, keyhe(q.z, q.x, q.w), t);
  }
}

// id-preserving growth (safe inside a round, after the filter): arrays are
// copied, the hash table is rebuilt from the live entries
static void grow_seg_records(gq_ctx* c, size_t cap) {
  Dev& D = c->D;
  size_t n = (size_t)c->hc.nsegrec;
  regrow(c, D.sg_uv, n, cap); regrow(c, D.sg_sid, n, cap); regrow(c, D.sg_fl, n, cap, 0);
  unsigned int h = pow2_at_least(2 * cap);
  dfree(D.sg_hk); dfree(D.sg_hv);
  D.sg_hk = dmalloc<unsigned long long>(h); D.sg_hv = dmalloc<int>(h); D.sg_hmask = h - 1;
  CK(cudaMemsetAsync(D.sg_hk, 0xff, (size_t)h * 8, c->st));
  if (n) LAUNCH(k_rehash_live_segs, n, D, (int)n);
  D.sgcap = (int)cap;
  realloc_owners(c);
  realloc_grid_nodes(c);
  if (g_trace) std::fprintf(stderr, "[grow] seg records cap %zu\n", cap);
}
static void grow_face_records(gq_ctx* c, size_t cap) {
  Dev& D = c->D;
  size_t n = (size_t)c->hc.nfacerec;
  regrow(c, D.sf_v, n, cap); regrow(c, D.sf_fl, n, cap, 0);
  unsigned int h = pow2_at_least(2 * cap);
  dfree(D.sf_hk); dfree(D.sf_hv);
  D.sf_hk = dmalloc<unsigned long long>(h); D.sf_hv = dmalloc<int>(h); D.sf_hmask = h - 1;
  CK(cudaMemsetAsync(D.sf_hk, 0xff, (size_t)h * 8, c->st));
  if (n) LAUNCH(k_rehash_live_faces, n, D, (int)n);
  D.sfcap = (int)cap;
  realloc_grid_nodes(c);
  if (g_trace) std::fprintf(stderr, "[grow] face records cap %zu\n", cap);
}
static void grow_t2(gq_ctx* c, size_t cap) {
  Dev& D = c->D;
  size_t n = (size_t)c->hc.nt2;
  regrow(c, D.t2v, n, cap); regrow(c, D.t2alive, n, cap, 0);
  dfree(c->T.own); c->T.own = dmalloc<int>(cap);
  CK(cudaMemsetAsync(c->T.own, 0x7f, cap * 4, c->st));
  unsigned int h = pow2_at_least(4 * cap);
  dfree(D.he_hk); dfree(D.he_hv);
  D.he_hk = dmalloc<unsigned long long>(h); D.he_hv = dmalloc<int>(h); D.he_hmask = h - 1;
  CK(cudaMemsetAsync(D.he_hk, 0xff, (size_t)h * 8, c->st));
  if (n) LAUNCH(k_t2_rehash_live, n, D, (int)n);
  D.t2cap = (int)cap;
  if (g_trace) std::fprintf(stderr, "[grow] 2D triangles cap %zu\n", cap);
}

// Before the insertions of a round (counts pulled): room for what `ni`
// inserted points (`nit` of them facet items) can create -- two subsegments
// per split, and a generous bound on the subfaces / 2D triangles of a fan.
static void ensure_round_room(gq_ctx* c, long long ni, long long nit) {
  Dev& D = c->D;
  long long sneed = c->hc.nsegrec + 2 * ni + 1024, fneed = c->hc.nfacerec + 32 * nit + 1024, tneed = c->hc.nt2 + 32 * nit + 1024;
  if (sneed > D.sgcap) grow_seg_records(c, std::max<size_t>(2 * (size_t)sneed, 2 * (size_t)D.sgcap));
  if (fneed > D.sfcap) grow_face_records(c, std::max<size_t>(2 * (size_t)fneed, 2 * (size_t)D.sfcap));
  if (tneed > D.t2cap) grow_t2(c, std::max<size_t>(2 * (size_t)tneed, 2 * (size_t)D.t2cap));
}

// Start of a round: drop dead records / 2D triangles when half the capacity
// is used (ids are renumbered: nothing outside the round keeps one), and grow
// when the live ones still fill a quarter.
static void maintain_seg_records(gq_ctx* c) {
  Dev& D = c->D;
  int n = c->hc.nsegrec;
  if ((size_t)n * 2 <= (size_t)D.sgcap) return;
  ensure_tmp(c, n + 1);
  LAUNCH(k_live_flags, n, D.sg_fl, n, c->tmpA);
  int live = scan_total(c, c->tmpA, c->tmpB, n);
  size_t cap = (size_t)D.sgcap;
  if ((size_t)live * 4 > cap) cap = std::max<size_t>(4 * (size_t)live, 2 * cap);
  int2* uv2 = dmalloc<int2>(cap); int* sid2 = dmalloc<int>(cap); unsigned int* fl2 = dmalloc<unsigned int>(cap);
  LAUNCH(k_move_seg_records, n, D, c->tmpA, c->tmpB, n, uv2, sid2, fl2);
  dfree(D.sg_uv); dfree(D.sg_sid); dfree(D.sg_fl);
  D.sg_uv = uv2; D.sg_sid = sid2; D.sg_fl = fl2;
  unsigned int h = pow2_at_least(2 * cap);
  if (h != D.sg_hmask + 1) { dfree(D.sg_hk); dfree(D.sg_hv); D.sg_hk = dmalloc<unsigned long long>(h); D.sg_hv = dmalloc<int>(h); D.sg_hmask = h - 1; }
  CK(cudaMemsetAsync(D.sg_hk, 0xff, (size_t)h * 8, c->st));
  if (live > 0) LAUNCH(k_rehash_segs, live, D, live);
  bool grew = cap != (size_t)D.sgcap;
  D.sgcap = (int)cap;
  c->hc.nsegrec = live;
  push(c);
  if (grew) { realloc_owners(c); realloc_grid_nodes(c); }
  if (g_trace) std::fprintf(stderr, "[grow] seg records %d -> %d live, cap %zu\n", n, live, cap);
}
static void maintain_face_records(gq_ctx* c) {
  Dev& D = c->D;
  int n = c->hc.nfacerec;
  if ((size_t)n * 2 <= (size_t)D.sfcap) return;
  ensure_tmp(c, n + 1);
  LAUNCH(k_live_flags, n, D.sf_fl, n, c->tmpA);
  int live = scan_total(c, c->tmpA, c->tmpB, n);
  size_t cap = (size_t)D.sfcap;
  if ((size_t)live * 4 > cap) cap = std::max<size_t>(4 * (size_t)live, 2 * cap);
  int4* v2 = dmalloc<int4>(cap); unsigned int* fl2 = dmalloc<unsigned int>(cap);
  LAUNCH(k_move_face_records, n, D, c->tmpA, c->tmpB, n, v2, fl2);
  dfree(D.sf_v); dfree(D.sf_fl);
  D.sf_v = v2; D.sf_fl = fl2;
  unsigned int h = pow2_at_least(2 * cap);
  if (h != D.sf_hmask + 1) { dfree(D.sf_hk); dfree(D.sf_hv); D.sf_hk = dmalloc<unsigned long long>(h); D.sf_hv = dmalloc<int>(h); D.sf_hmask = h - 1; }
  CK(cudaMemsetAsync(D.sf_hk, 0xff, (size_t)h * 8, c->st));
  if (live > 0) LAUNCH(k_rehash_faces, live, D, live);
  bool grew = cap != (size_t)D.sfcap;
  D.sfcap = (int)cap;
  c->hc.nfacerec = live;
  push(c);
  if (grew) realloc_grid_nodes(c);
  if (g_trace) std::fprintf(stderr, "[grow] face records %d -> %d live, cap %zu\n", n, live, cap);
}
// facet 2D triangles (alive ones keep their relative order)
static void maintain_t2(gq_ctx* c) {
  Dev& D = c->D;
  int n = c->hc.nt2;
  if ((size_t)n * 2 <= (size_t)D.t2cap) return;
  ensure_tmp(c, n + 1);
  LAUNCH(k_t2_live, n, D, n, c->tmpA);
  int live = scan_total(c, c->tmpA, c->tmpB, n);
  size_t cap = (size_t)D.t2cap;
  if ((size_t)live * 4 > cap) cap = std::max<size_t>(4 * (size_t)live, 2 * cap);
  int4* v2 = dmalloc<int4>(cap);
  LAUNCH(k_t2_move, n, D, c->tmpA, c->tmpB, n, v2);
  LAUNCH(k_t2_last_remap, std::max(D.npoly, 1), D, c->tmpA, c->tmpB);
  dfree(D.t2v);
  D.t2v = v2;
  if (cap != (size_t)D.t2cap) {
    dfree(D.t2alive); D.t2alive = dmalloc<uint8_t>(cap);
    dfree(c->T.own); c->T.own = dmalloc<int>(cap);
    CK(cudaMemsetAsync(c->T.own, 0x7f, cap * 4, c->st));
  }
  CK(cudaMemsetAsync(D.t2alive, 0, cap, c->st));
  if (live > 0) CK(cudaMemsetAsync(D.t2alive, 1, (size_t)live, c->st));
  unsigned int h = pow2_at_least(4 * cap);
  if (h != D.he_hmask + 1) { dfree(D.he_hk); dfree(D.he_hv); D.he_hk = dmalloc<unsigned long long>(h); D.he_hv = dmalloc<int>(h); D.he_hmask = h - 1; }
  CK(cudaMemsetAsync(D.he_hk, 0xff, (size_t)h * 8, c->st));
  if (live > 0) LAUNCH(k_t2_rehash, live, D, live);
  D.t2cap = (int)cap;
  c->hc.nt2 = live;
  push(c);
  if (g_trace) std::fprintf(stderr, "[grow] 2D triangles %d -> %d live, cap %zu\n", n, live, cap);
}
// start of a round (counters pulled): vertices / tets with a round's worth of
// headroom, records and 2D triangles compacted / grown when half full
static void maintain_capacity(gq_ctx* c) {
  long long nv = c->hc.nv, nt = c->hc.nt;
  ensure_mesh_room(c, nv + std::max(nv / 2, 65536LL), nt + std::max(nt / 2, 1LL << 20));
  maintain_seg_records(c);
  maintain_face_records(c);
  maintain_t2(c);
}
