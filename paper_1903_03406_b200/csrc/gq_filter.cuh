// gq_filter.cuh -- conflict filter: local-minimum iterations == greedy_oracle (growblast.py:123-207).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

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

__global__ void k_claim(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 0) continue;
    int r = C.rank[c];
    for_claims(D, C, W, c, [&](int k) { atomicMin(W.own + k, r); });
  }
}
__global__ void k_decide(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, int n, int it) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 0) continue;
    int r = C.rank[c];
    bool win = true;
    for_claims(D, C, W, c, [&](int k) { if (W.own[k] != r) win = false; });
    if (win) C.state[c] = 10 + it;   // accepted this iteration (marked next)
  }
}
__global__ void k_mark(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, int n, int it) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 10 + it) continue;
    for_claims(D, C, W, c, [&](int k) { W.own[k] = -1; });
    C.state[c] = 1;
  }
}
__global__ void k_reject(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, int n, int* undecided) {
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
// grid-wide barrier of the cooperative launch, or the block barrier when the
// kernel runs as one block (small rounds: no cooperative launch, which would
// serialise against the other contexts' work on the device)
template <bool ONE>
__device__ __forceinline__ void gsync() {
  if (ONE) __syncthreads(); else cg::this_grid().sync();
}
template <bool ONE>
__global__ void __launch_bounds__(256) k_filter_coop(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, int n, int* ctr) {
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
    gsync<ONE>();
    for (int c = gw; c < n; c += nw) {                       // decide
      if (C.state[c] != 0) continue;
      const int r = C.rank[c];
      bool win = true;
      warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] != r) win = false; });
      win = __all_sync(FULL, win);
      if (win && lane == 0) C.state[c] = 10 + it;
    }
    gsync<ONE>();
    for (int c = gw; c < n; c += nw) {                       // mark
      if (C.state[c] != 10 + it) continue;
      warp_claims(D, C, W, c, lane, [&](int k) { W.own[k] = -1; });
      __syncwarp();
      if (lane == 0) C.state[c] = 1;
    }
    gsync<ONE>();
    int und = 0;
    for (int c = gw; c < n; c += nw) {                       // reject
      if (C.state[c] != 0) continue;
      bool hit = false;
      warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] == -1) hit = true; });
      hit = __any_sync(FULL, hit);
      if (lane == 0) { if (hit) C.state[c] = 4; else ++und; }
    }
    if (lane == 0 && und) atomicAdd(ctr + it % 3, und);
    gsync<ONE>();
    for (int c = gw; c < n; c += nw) {                       // release the claims of losers
      const int st = C.state[c];
      if (st != 0 && st != 4) continue;
      warp_claims(D, C, W, c, lane, [&](int k) { if (W.own[k] >= 0) W.own[k] = INT_MAX; });
      __syncwarp();
      if (st == 4 && lane == 0) C.state[c] = 2;
    }
    gsync<ONE>();
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
__global__ void k_strict_state(const __grid_constant__ Cand C, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (C.state[c] == 10) C.state[c] = 1;
    else if (C.state[c] == 0) C.state[c] = 2;
}
__global__ void k_reset_claims(const __grid_constant__ Dev D, const __grid_constant__ Cand C, Owners W, int n, int all) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    int s = C.state[c];
    if (!all && s != 0 && s != 2) continue;
    if (all && (s < 0 || s == 3)) continue;
    for_claims(D, C, W, c, [&](int k) { if (all || W.own[k] >= 0) W.own[k] = INT_MAX; });
  }
}

