// gq_check.cuh -- post-round constraint verification (refine.py:549-571, 816-858).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

// ---------------------------------------------------------------------------
// constraint verification (refine.py:549-571, 829-851), mesh-local:
// a subsegment is tested against the vertices of the tets around it, a
// subface against the apexes of its two tets (identical to the
// reference's global KD-tree scans).
// distance of p from the line (u,v) / plane (a,b,c), relative to the element
// size: diagnostics only (which verification outcome fired)
__device__ inline bool near_line(const double* u, const double* v, const double* p) {
  double d[3] = {v[0] - u[0], v[1] - u[1], v[2] - u[2]}, w[3] = {p[0] - u[0], p[1] - u[1], p[2] - u[2]};
  double cx = d[1] * w[2] - d[2] * w[1], cy = d[2] * w[0] - d[0] * w[2], cz = d[0] * w[1] - d[1] * w[0];
  double l2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  return (cx * cx + cy * cy + cz * cz) < 1e-16 * l2 * l2;
}
__device__ inline bool near_plane(const double* a, const double* b, const double* c, const double* p) {
  double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  double h = n[0] * (p[0] - a[0]) + n[1] * (p[1] - a[1]) + n[2] * (p[2] - a[2]);
  double n2 = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
  double s2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  return h * h < 1e-16 * n2 * s2;
}
__device__ __noinline__ bool seg_check(const Dev& D, int r, Scratch& S) {   // true -> encroached or missing
  int2 e = D.sg_uv[r];
  const double *pu = PT(D, e.x), *pv = PT(D, e.y);
  bool present = false, enc = false;
  int ew = -1;
  around_vertex(D, e.x, S.tset, S.stack, 2 * S.cap, [&](int t) {
    int4 q = D.tv[t];
    if (!has_v(q, e.y)) return false;
    present = true;
    for (int k = 0; k < 4; ++k) {
      int w = tvk(q, k);
      if (w == GHOST || w == e.x || w == e.y) continue;
      if (encroaches_segment(pu, pv, PT(D, w))) { enc = true; ew = w; return true; }
    }
    return false;
  });
  if (!present) atomicAdd(&D.ctr->chk[0], 1u);
  else if (enc) atomicAdd(&D.ctr->chk[near_line(pu, pv, PT(D, ew)) ? 2 : 1], 1u);
  return !present || enc;
}
__device__ __noinline__ bool face_check(const Dev& D, int r, Scratch& S) {
  int4 f = D.sf_v[r];
  int slot = find_face(D, f.x, f.y, f.z, S.tset, S.stack, 2 * S.cap);
  if (slot < 0) { atomicAdd(&D.ctr->chk[3], 1u); return true; }
  const double *a = PT(D, f.x), *b = PT(D, f.y), *c = PT(D, f.z);
  int t = slot >> 2, i = slot & 3;
  int w = tvk(D.tv[t], i);
  if (w != GHOST && encroaches_face(a, b, c, PT(D, w))) {
    atomicAdd(&D.ctr->chk[near_plane(a, b, c, PT(D, w)) ? 5 : 4], 1u);
    return true;
  }
  int nb = tnk(D, t, i);
  int u = nb >> 2, j = nb & 3;
  int w2 = tvk(D.tv[u], j);
  if (w2 != GHOST && encroaches_face(a, b, c, PT(D, w2))) {
    atomicAdd(&D.ctr->chk[near_plane(a, b, c, PT(D, w2)) ? 5 : 4], 1u);
    return true;
  }
  return false;
}
// mode 0: records flagged CHECK; mode 1: every live record (full_verify)
__global__ void k_check(const __grid_constant__ Dev D, const __grid_constant__ Scr SC, int mode, int* found) {
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
__global__ void k_clear_flag(const __grid_constant__ Dev D, unsigned int flag) {
  int ns = D.ctr->nsegrec, nf = D.ctr->nfacerec;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < ns + nf; w += gridDim.x * blockDim.x) {
    if (w < ns) D.sg_fl[w] &= ~flag; else D.sf_fl[w - ns] &= ~flag;
  }
}
// counts: [0] pending segs, [1] pending faces, [2] enc segs (live), [3] enc faces
__global__ void k_count_pending(const __grid_constant__ Dev D, int* out) {
  int ns = D.ctr->nsegrec, nf = D.ctr->nfacerec;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < ns + nf; w += gridDim.x * blockDim.x) {
    unsigned int f = w < ns ? D.sg_fl[w] : D.sf_fl[w - ns];
    if (!(f & RF_LIVE) || !(f & RF_ENC)) continue;
    int base = w < ns ? 0 : 1;
    atomicAdd(out + 2 + base, 1);
    if (!(f & RF_BLOCK) && !(f & RF_SKIP)) atomicAdd(out + base, 1);
  }
}
__global__ void k_flag_pending_keys(const __grid_constant__ Dev D, int phase, unsigned int need, unsigned int deny, int* flags,
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
__global__ void k_face_a(const __grid_constant__ Dev D, const int* recs, int n, unsigned int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = (unsigned int)D.sf_v[recs[i]].x;
}
__global__ void k_flag_bad(const __grid_constant__ Dev D, double B, int* flags) {
  int nt = D.ctr->nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x)
    flags[t] = D.alive[t] == 1 && D.tv[t].w >= 0 && D.ratio[t] > B && D.skip[t] == 0;
}
__global__ void k_set_cands(const __grid_constant__ Cand C, int n0, int n, int kind, const int* tgts, int pool0) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    C.kind[n0 + k] = kind; C.tgt[n0 + k] = tgts[k]; C.pool[n0 + k] = pool0 + k;
    C.status[n0 + k] = CS_OK; C.bigi[n0 + k] = -1;
  }
}
__global__ void k_clear_redir(const __grid_constant__ Dev D, int phase) {
  int n = phase == 0 ? D.ctr->nsegrec : D.ctr->nfacerec;
  unsigned int* fl = phase == 0 ? D.sg_fl : D.sf_fl;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) fl[r] &= ~RF_REDIR;
}

