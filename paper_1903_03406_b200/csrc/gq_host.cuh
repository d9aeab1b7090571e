// gq_host.cuh -- host driver: context, caching allocator, capacities, rounds (refine.py:523-925).
// Part of the single translation unit gq_main.cu (included in order).
#pragma once

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
// A context's calls use the context's own cache (set by CtxScope for the
// duration of each C-ABI call), so blocks freed by one context's stream are
// never handed to another context's concurrently running stream.  Calls
// without a context (gq_batch) use a per-device cache.
static thread_local DevCache* tl_cache = nullptr;
static DevCache& dev_cache() {
  if (tl_cache) return *tl_cache;
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
  DevCache cache;
  char* pin = nullptr; size_t pin_cap = 0, pin_used = 0;                 // pinned read-back staging
  unsigned long long errn0 = 0;                                           // device error count at the call's start
  std::vector<std::tuple<void*, size_t, size_t>> staged;
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
  int4* tvn2 = nullptr; uint8_t *sub2 = nullptr, *seg2 = nullptr, *skip2 = nullptr; double* ratio2 = nullptr;
  struct QBuf { int *a, *b, *c, *d, *e, *f, *g, *h; size_t cap; } Q{};
  HugeArena HA{};            // global-memory block storage of the huge region tier
  int* hlist = nullptr; size_t hlist_cap = 0;
  bool allocated = false;
};

struct CtxScope {   // binds the calling thread's allocations to a context's cache
  DevCache* prev;
  explicit CtxScope(gq_ctx* c) : prev(tl_cache) { tl_cache = &c->cache; }
  ~CtxScope() { tl_cache = prev; }
};

static double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static thread_local double g_prof[8];
// fine stage timers (GQ_PROFILE=2): synchronise and charge the elapsed time
static thread_local bool g_trace = false;
// Experiment / debug switches, read once when the library loads (never on the
// per-round path)
static const bool o_thread_regions = getenv("GQ_THREAD_REGIONS") != nullptr;
static const bool o_filter_launches = getenv("GQ_FILTER_LAUNCHES") != nullptr;
static const bool o_thread_init = getenv("GQ_THREAD_INIT") != nullptr;
static const bool o_init_launches = getenv("GQ_INIT_LAUNCHES") != nullptr;
static const bool o_fallback_serial = getenv("GQ_FALLBACK_SERIAL") != nullptr;   // one-thread fallback loop (comparisons)
static const int o_fb_window = getenv("GQ_FB_WINDOW") ? std::max(1, atoi(getenv("GQ_FB_WINDOW"))) : 1024;   // fallback wave window
static const int o_trace_from = getenv("GQ_TRACE_FROM") ? atoi(getenv("GQ_TRACE_FROM")) : -1;
static const bool g_grid_thread = getenv("GQ_GRID_THREAD") != nullptr;   // experiments: thread-per-query grid kernels
static thread_local bool g_fine = false;      // GQ_PROFILE=2: host clock after a sync per stage
static thread_local bool g_fine_ev = false;   // GQ_PROFILE=3: events per stage (device timeline, no syncs)
static thread_local double g_fine_t[40];
static const char* g_fine_names[40] = {"i.region", "i.big", "i.filter", "i.scan", "i.kill", "i.stars", "i.compact",
  "p.gridsync", "p.newverts", "p.check", "p.compact", "r.sorted", "r.make", "r.redirect", "r.append", "f.states",
  "f.rank", "f.lfmis", "x.acc", "x.ids", "x.star", "x.postins", "i.misc", "r.misc", "g.warp", "g.ovfscan", "g.block",
  "r.setup", "r.gridc", "r.kept", "x.fallback", "r.misc2", "x.verts", "x.items", "x.t2"};
static thread_local double g_fine_last = 0;
static void fine(gq_ctx* c, int k);
// Device -> host reads go through a pinned staging buffer on the context's
// stream: a pageable destination makes the copy synchronous and serialises it
// against every other context's stream (C5 runs several at once).  stage()
// enqueues, sync() waits and delivers.
static void stage(gq_ctx* c, void* dst, const void* src, size_t bytes) {
  if (c->pin_used + bytes + 64 > c->pin_cap) {
    if (!c->staged.empty()) {                     // no room beside pending reads: pageable copy
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->st));
      return;
    }
    size_t cap = c->pin_cap;                      // nothing pending: grow the staging buffer
    while (bytes + 64 > cap) cap *= 2;
    CK(cudaFreeHost(c->pin));
    c->pin = nullptr;
    CK(cudaHostAlloc((void**)&c->pin, cap, cudaHostAllocDefault));
    c->pin_cap = cap;
  }
  size_t off = c->pin_used;
  CK(cudaMemcpyAsync(c->pin + off, src, bytes, cudaMemcpyDeviceToHost, c->st));
  c->staged.push_back({dst, off, bytes});
  c->pin_used = (off + bytes + 15) & ~size_t(15);
}
static void sync(gq_ctx* c) {
  // the error word travels with the stream too (cudaMemcpyFromSymbol would use the legacy stream)
  const size_t eoff = c->pin_cap - 16;
  CK(cudaMemcpyFromSymbolAsync(c->pin + eoff, g_errn, sizeof(unsigned long long), 0, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyFromSymbolAsync(c->pin + eoff + 8, g_err, sizeof(unsigned int), 0, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (auto& s : c->staged) std::memcpy(std::get<0>(s), c->pin + std::get<1>(s), std::get<2>(s));
  c->staged.clear();
  c->pin_used = 0;
  unsigned long long n = 0;
  unsigned int e = 0;
  std::memcpy(&n, c->pin + eoff, sizeof(n));
  std::memcpy(&e, c->pin + eoff + 8, sizeof(e));
  if (n != c->errn0) {
    c->errn0 = n;   // reported once; the next call starts from here
    char buf[128];
    std::snprintf(buf, sizeof buf, "device error flags 0x%x", e);
    throw std::runtime_error(buf);
  }
}
// error baseline of a call (after the stream's earlier work)
static void err_baseline(gq_ctx* c) {
  CK(cudaMemcpyFromSymbolAsync(&c->errn0, g_errn, sizeof(unsigned long long), 0, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
}
static void pull(gq_ctx* c) { stage(c, &c->hc, c->dctr, sizeof(Counters)); sync(c); }
// the mesh / record counts only: the instrumentation counters are device-owned
static void push(gq_ctx* c) { CK(cudaMemcpyAsync(c->dctr, &c->hc, offsetof(Counters, region_calls), cudaMemcpyHostToDevice, c->st)); }
static int grid_for(long long n, int bs = 128, int cap = 148 * 16) {
  long long g = (n + bs - 1) / bs;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}
#define LAUNCH(kern, n, ...) do { kern<<<grid_for(n), 128, 0, c->st>>>(__VA_ARGS__); c->launches++; CK(cudaGetLastError()); } while (0)
// one item per warp (lane 0), scratch slot per warp
#define LAUNCH_W(kern, n, ...) do { kern<<<std::max(1, (int)((std::min<long long>(n, c->S.nthreads) + 3) / 4)), 128, 0, c->st>>>(__VA_ARGS__); c->launches++; CK(cudaGetLastError()); } while (0)
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
  stage(c, &last_f, flags + n - 1, 4);
  stage(c, &last_s, c->tmpC + n - 1, 4);
  sync(c);
  return last_f + last_s;
}
static void exclusive_scan(gq_ctx* c, const int* in, int* out, int n) {
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n, c->st);
  ensure_cub(c, need);
  cub::DeviceScan::ExclusiveSum(c->cub_tmp, need, in, out, n, c->st);
}
// device -> host copy ordered on the context's stream, complete on return
static void d2h(gq_ctx* c, void* dst, const void* src, size_t bytes) {
  stage(c, dst, src, bytes);
  sync(c);
}
static int read_int(gq_ctx* c, const int* d) { int v; stage(c, &v, d, sizeof v); sync(c); return v; }

static void alloc_scratch(Scr& s, int nthreads, int cap, int tcap, int fcap, cudaStream_t st) {
  s.nthreads = nthreads; s.cap = cap; s.tcap = tcap; s.fcap = fcap;
  s.tkey = dmalloc<int>((size_t)nthreads * tcap); s.tval = dmalloc<int>((size_t)nthreads * tcap);
  s.tep = dmalloc<unsigned int>((size_t)nthreads * tcap);
  s.fkey = dmalloc<unsigned long long>((size_t)nthreads * fcap); s.fep = dmalloc<unsigned int>((size_t)nthreads * fcap);
  s.epoch = dmalloc<unsigned int>((size_t)nthreads * 2);
  CK(cudaMemsetAsync(s.tep, 0, (size_t)nthreads * tcap * 4, st)); CK(cudaMemsetAsync(s.fep, 0, (size_t)nthreads * fcap * 4, st));
  CK(cudaMemsetAsync(s.epoch, 0, (size_t)nthreads * 2 * 4, st));
  s.list = dmalloc<int>((size_t)nthreads * cap); s.stack = dmalloc<int>((size_t)nthreads * cap * 2);
  s.in = dmalloc<uint8_t>((size_t)nthreads * cap); s.comp = dmalloc<uint8_t>((size_t)nthreads * cap);
}

static void alloc_cands(gq_ctx* c, int cap, int bigcap) {
  Cand& C = c->C;
  C.cap = cap;
  C.segpoly = c->D.segpoly;
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
static void copy_huge(Cand& d, const Cand& s) {
  d.htets = s.htets; d.hbf = s.hbf; d.hcr = s.hcr; d.hcrf = s.hcrf; d.hbsub = s.hbsub; d.hbseg = s.hbseg;
  d.heseg = s.heseg; d.hskey = s.hskey; d.hsv0 = s.hsv0; d.hsv1 = s.hsv1;
  d.nhugecap = s.nhugecap; d.ht = s.ht; d.hf = s.hf; d.hc = s.hc; d.hs = s.hs;
}
static void free_cands(Cand& C) {
  void* ps[] = {C.kind, C.tgt, C.seed, C.status, C.memb, C.pool, C.rank, C.allow, C.nallow, C.extra, C.p, C.h, C.canon,
                C.state, C.vid, C.nt0, C.ntet, C.nbf, C.ncr, C.nbsub, C.nbseg, C.neseg, C.mind, C.tets, C.bf, C.cr,
                C.crf, C.bsub, C.bseg, C.eseg, C.rseg, C.rface, C.nrseg, C.nrface, C.bigi, C.btets, C.bbf, C.bcr,
                C.bcrf, C.bbsub, C.bbseg, C.beseg};
  for (void* p : ps) if (p) dfree(p);
  Cand keep = C;       // the huge slabs are owned by ensure_huge / free_huge
  C = Cand{};
  copy_huge(C, keep);
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
  copy_huge(c->C, old);
  alloc_cands(c, std::max(need, 2 * old.cap), old.nbigcap);
  Cand& C = c->C;
  size_t k = (size_t)n_keep;
#define CPY(f, w) CK(cudaMemcpyAsync(C.f, old.f, sizeof(*old.f) * (w) * k, cudaMemcpyDeviceToDevice, c->st))
  CPY(kind, 1); CPY(tgt, 1); CPY(seed, 1); CPY(status, 1); CPY(memb, 1); CPY(pool, 1); CPY(rank, 1);
  CPY(allow, 1); CPY(nallow, 1); CPY(extra, 1); CPY(p, 3); CPY(h, 1); CPY(canon, 1); CPY(state, 1);
  CPY(vid, 1); CPY(nt0, 1); CPY(ntet, 1); CPY(nbf, 1); CPY(ncr, 1); CPY(nbsub, 1); CPY(nbseg, 1);
  CPY(neseg, 1); CPY(mind, 1); CPY(tets, CT); CPY(bf, CF); CPY(cr, CC); CPY(crf, CC); CPY(bsub, CC);
  CPY(bseg, CC); CPY(eseg, CC); CPY(rseg, CRD); CPY(rface, CRD); CPY(nrseg, 1); CPY(nrface, 1); CPY(bigi, 1);
#undef CPY
  size_t kb = (size_t)old.nbigcap;
  CK(cudaMemcpyAsync(C.btets, old.btets, 4 * kb * CTB, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(C.bbf, old.bbf, 4 * kb * CFB, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(C.bcr, old.bcr, 4 * kb * CCB, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(C.bcrf, old.bcrf, 4 * kb * CCB, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(C.bbsub, old.bbsub, 4 * kb * CCB, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(C.bbseg, old.bbseg, 4 * kb * CCB, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(C.beseg, old.beseg, 4 * kb * CCB, cudaMemcpyDeviceToDevice, c->st));
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
    if (keep) CK(cudaMemcpyAsync(q, ptr, 4 * keep * w, cudaMemcpyDeviceToDevice, c->st));
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
  double capx = getenv("GQ_CAPX") ? atof(getenv("GQ_CAPX")) : 1.0;   // experiments: capacity multiplier
  // (the minimums cover bulk construction and the initial constraints; the
  // rounds grow everything on demand, gq_grow.cuh)
  size_t vcap = std::max<size_t>((size_t)(capx * (65536 + (size_t)n * 8)), (size_t)n + 1024);
  size_t tcap = std::max<size_t>((size_t)(capx * std::max<size_t>(1 << 21, (size_t)n * 64)), (size_t)n * 40 + 65536);
  D.vcap = (int)vcap; D.tcap = (int)tcap;
  D.P = dmalloc<double>(3 * vcap); D.vorigin = dmalloc<uint8_t>(vcap); D.vert_tet = dmalloc<int>(vcap);
  D.vsid = dmalloc<int>(vcap);
  D.tv.p = dmalloc<int4>(2 * tcap); D.tn.p = D.tv.p + 1; D.alive = dmalloc<uint8_t>(tcap);
  D.sub = dmalloc<uint8_t>(tcap); D.seg = dmalloc<uint8_t>(tcap); D.skip = dmalloc<uint8_t>(tcap);
  D.ratio = dmalloc<double>(tcap);
  CK(cudaMemsetAsync(D.alive, 0, tcap, c->st));
  if (getenv("GQ_PROFILE")) std::fprintf(stderr, "[gq] capacities: verts %zu tets %zu\n", vcap, tcap);
  size_t sgcap = std::max<size_t>((size_t)(capx * (65536 + (size_t)m * 32 + vcap / 8)), (size_t)m + 1024);
  D.sgcap = (int)sgcap;
  D.sg_uv = dmalloc<int2>(sgcap); D.sg_sid = dmalloc<int>(sgcap); D.sg_fl = dmalloc<unsigned int>(sgcap);
  unsigned int sgh = pow2_at_least(2 * sgcap);
  D.sg_hk = dmalloc<unsigned long long>(sgh); D.sg_hv = dmalloc<int>(sgh); D.sg_hmask = sgh - 1;
  CK(cudaMemsetAsync(D.sg_hk, 0xff, (size_t)sgh * 8, c->st));
  size_t sfcap = std::max<size_t>((size_t)(capx * (65536 + (size_t)npidx * 32 + vcap)), (size_t)npidx + 1024);
  D.sfcap = (int)sfcap;
  D.sf_v = dmalloc<int4>(sfcap); D.sf_fl = dmalloc<unsigned int>(sfcap);
  unsigned int sfh = pow2_at_least(2 * sfcap);
  D.sf_hk = dmalloc<unsigned long long>(sfh); D.sf_hv = dmalloc<int>(sfh); D.sf_hmask = sfh - 1;
  CK(cudaMemsetAsync(D.sf_hk, 0xff, (size_t)sfh * 8, c->st));
  size_t t2cap = std::max<size_t>((size_t)(capx * (65536 + (size_t)npidx * 8 + 2 * vcap)), 2 * (size_t)npidx + 1024);
  D.t2cap = (int)t2cap;
  D.t2v = dmalloc<int4>(t2cap); D.t2alive = dmalloc<uint8_t>(t2cap);
  CK(cudaMemsetAsync(D.t2alive, 0, t2cap, c->st));
  unsigned int heh = pow2_at_least(4 * t2cap);
  D.he_hk = dmalloc<unsigned long long>(heh); D.he_hv = dmalloc<int>(heh); D.he_hmask = heh - 1;
  CK(cudaMemsetAsync(D.he_hk, 0xff, (size_t)heh * 8, c->st));
  D.t2count = dmalloc<int>(std::max(f, 1));
  CK(cudaMemsetAsync(D.t2count, 0, std::max(f, 1) * 4, c->st));
  D.poly_keep = dmalloc<int2>(std::max(f, 1));
  D.poly_obl = dmalloc<uint8_t>(std::max(f, 1));
  D.poly_convex = dmalloc<uint8_t>(std::max(f, 1));
  CK(cudaMemsetAsync(D.poly_convex, 1, std::max(f, 1), c->st));
  D.poly_off = nullptr; D.poly_idx = nullptr;
  D.t2last = dmalloc<int>(std::max(f, 1));
  CK(cudaMemsetAsync(D.t2last, 0xff, 4 * (size_t)std::max(f, 1), c->st));
  D.segpoly_off = dmalloc<int>(m + 1);
  D.segpoly = dmalloc<int>(std::max(npidx, 1));
  D.sid_uv = dmalloc<int2>(std::max(m, 1));
  D.vapex = nullptr;   // set by refine_impl
  D.poly_obl_hull = 0;
  D.nsid = m; D.npoly = f;
  c->dctr = dmalloc<Counters>(1);
  D.ctr = c->dctr;
  // large vertex-star arenas (around_vertex overflow path)
  D.vp_n = 64; D.vp_cap = 1 << 17;
  {
    size_t nb = (size_t)D.vp_n * D.vp_cap;
    D.vp_key = dmalloc<int>(nb); D.vp_val = dmalloc<int>(nb); D.vp_ep = dmalloc<unsigned int>(nb);
    D.vp_stack = dmalloc<int>(nb); D.vp_epoch = dmalloc<unsigned int>(D.vp_n); D.vp_lock = dmalloc<int>(D.vp_n);
    CK(cudaMemsetAsync(D.vp_ep, 0, 4 * nb, c->st));
    CK(cudaMemsetAsync(D.vp_epoch, 0, 4 * (size_t)D.vp_n, c->st));
    CK(cudaMemsetAsync(D.vp_lock, 0, 4 * (size_t)D.vp_n, c->st));
  }
  // filter owners: [tets | faces | seg records]
  c->W.toff = 0; c->W.foff = (int)tcap; c->W.soff = (int)(5 * tcap);
  c->W.own = dmalloc<int>(5 * tcap + sgcap);
  CK(cudaMemsetAsync(c->W.own, 0x7f, (5 * tcap + sgcap) * 4, c->st));
  // 2D items
  c->T.cap = T2_CAP; c->T.rcap = T2_CAP;
  static_assert(T2_CAP <= CT * 2, "tri2_cavity: DFS stack + component marks (2 * T2_CAP) must fit the 2 * Scratch.cap stack");
  c->T.icap = 0;
  c->T.cand = c->T.pid = c->T.state = c->T.ncav = c->T.nrem = c->T.cav = c->T.rem = nullptr;   // freed by free_all
  ensure_items(c, 1 << 16);
  c->T.own = dmalloc<int>(t2cap);
  CK(cudaMemsetAsync(c->T.own, 0x7f, t2cap * 4, c->st));
  c->L.cap = 1 << 20; c->L.rows = dmalloc<int>((size_t)SKIP_ROW * c->L.cap);
  c->d_int = dmalloc<int>(64);
  alloc_scratch(c->S, 16384, CT * 2, 1024, 2048, c->st);
  alloc_scratch(c->SB, 512, CTB * 2, 32768, 32768, c->st);
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

static void free_huge(gq_ctx* c);
static void free_all(gq_ctx* c) {
  if (!c->allocated) return;
  Dev& D = c->D;
  void* ps[] = {D.P, D.vorigin, D.vert_tet, D.vsid, D.tv.p, D.alive, D.sub, D.seg, D.skip, D.ratio, D.sg_uv,
                D.sg_sid, D.sg_fl, D.sg_hk, D.sg_hv, D.sf_v, D.sf_fl, D.sf_hk, D.sf_hv, D.t2v, D.t2alive, D.he_hk,
                D.he_hv, D.t2count, D.poly_keep, D.poly_obl, D.t2last, D.segpoly_off, D.segpoly, D.sid_uv, D.vapex, D.poly_convex, (void*)D.poly_off, (void*)D.poly_idx, D.vp_key, D.vp_val, D.vp_ep, D.vp_stack, D.vp_epoch, D.vp_lock, c->dctr, c->W.own, c->T.cand,
                c->T.pid, c->T.state, c->T.cav, c->T.ncav, c->T.rem, c->T.nrem, c->T.own, c->L.rows, c->d_int,
                c->S.tkey, c->S.tval, c->S.tep, c->S.fkey, c->S.fep, c->S.epoch, c->S.list, c->S.stack, c->S.in,
                c->S.comp, c->SB.tkey, c->SB.tval, c->SB.tep, c->SB.fkey, c->SB.fep, c->SB.epoch, c->SB.list,
                c->SB.stack, c->SB.in, c->SB.comp, c->tmpA, c->tmpB, c->tmpC, c->k64a, c->k64b, c->k32a, c->k32b,
                c->cub_tmp, c->d_order, c->G.start, c->G.codes, c->G.cnt, c->G.nbig, c->Q.a, c->Q.b, c->Q.c,
                c->Q.d, c->Q.e, c->Q.f, c->Q.g, c->Q.h, c->tvn2, c->sub2, c->seg2, c->skip2, c->ratio2};
  for (void* p : ps) if (p) dfree(p);
  free_huge(c);
  free_cands(c->C);
  c->allocated = false;
  c->tmpcap = 0; c->cub_cap = 0; c->cub_tmp = nullptr;
  c->tmpA = c->tmpB = c->tmpC = nullptr; c->k64a = c->k64b = nullptr; c->k32a = c->k32b = nullptr; c->d_order = nullptr;
  c->Q = {};
  c->tvn2 = nullptr; c->sub2 = c->seg2 = c->skip2 = nullptr; c->ratio2 = nullptr;
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
// huge region tier: slabs (ht tets each) for n candidates and block storage
static void free_huge(gq_ctx* c) {
  Cand& C = c->C;
  void* ps[] = {C.htets, C.hbf, C.hcr, C.hcrf, C.hbsub, C.hbseg, C.heseg, C.hskey, C.hsv0, C.hsv1,
                c->HA.hkey, c->HA.hval, c->HA.cav, c->HA.f0, c->HA.f1, c->HA.in, c->HA.comp, c->HA.fkey, c->HA.fep,
                c->HA.fepoch, c->hlist};
  for (void* p : ps) if (p) dfree(p);
  C.htets = C.hbf = C.hcr = C.hcrf = C.hbsub = C.hbseg = C.heseg = nullptr;
  C.hskey = nullptr; C.hsv0 = C.hsv1 = nullptr; C.nhugecap = 0; C.ht = 0;
  c->HA = HugeArena{};
  c->hlist = nullptr; c->hlist_cap = 0;
}
static void ensure_huge(gq_ctx* c, int n, int mcap) {
  Cand& C = c->C;
  if (n <= C.nhugecap && mcap == C.ht) return;
  free_huge(c);
  int cap = std::max(n, 4);
  C.nhugecap = cap; C.ht = mcap; C.hf = 2 * mcap + 1024; C.hc = mcap / 4 + 256;
  C.hs = (int)pow2_at_least(4 * (size_t)C.hf);
  size_t k = (size_t)cap;
  C.htets = dmalloc<int>(k * C.ht); C.hbf = dmalloc<int>(k * C.hf);
  C.hcr = dmalloc<int>(k * C.hc); C.hcrf = dmalloc<int>(k * C.hc); C.hbsub = dmalloc<int>(k * C.hc);
  C.hbseg = dmalloc<int>(k * C.hc); C.heseg = dmalloc<int>(k * C.hc);
  C.hskey = dmalloc<unsigned long long>(k * C.hs); C.hsv0 = dmalloc<int>(k * C.hs); C.hsv1 = dmalloc<int>(k * C.hs);
  HugeArena& H = c->HA;
  H.nblocks = std::min(cap, 64);
  H.mcap = mcap; H.hcap = (int)pow2_at_least(2 * (size_t)mcap); H.fcap = (int)pow2_at_least(4 * (size_t)C.hf);
  size_t nb = (size_t)H.nblocks;
  H.hkey = dmalloc<int>(nb * H.hcap); H.hval = dmalloc<int>(nb * H.hcap);
  H.cav = dmalloc<int>(nb * H.mcap); H.f0 = dmalloc<int>(nb * H.mcap); H.f1 = dmalloc<int>(nb * H.mcap);
  H.in = dmalloc<uint8_t>(nb * H.mcap); H.comp = dmalloc<int>(nb * H.mcap);
  H.fkey = dmalloc<unsigned long long>(nb * H.fcap); H.fep = dmalloc<unsigned int>(nb * H.fcap);
  H.fepoch = dmalloc<unsigned int>(nb);
  CK(cudaMemsetAsync(H.fep, 0, 4 * nb * H.fcap, c->st));
  CK(cudaMemsetAsync(H.fepoch, 0, 4 * nb, c->st));
  c->hlist = dmalloc<int>(k); c->hlist_cap = k;
}
__global__ void k_status_of(const __grid_constant__ Cand C, const int* list, int n, int* out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = C.status[list[k]];
}
__global__ void k_set_status(const __grid_constant__ Cand C, const int* list, int n, int from, int to) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    if (C.status[list[k]] == from) C.status[list[k]] = to;
}
__global__ void k_mark_memb(const __grid_constant__ Cand C, const int* list, int n, int status, int memb) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    if (C.status[list[k]] == status) C.memb[list[k]] = memb;
}
// block-tier overflows of this round: the huge tier, capacities doubled until
// every cavity fits (64k tets at most: beyond, the candidate fails).  Cavities
// that large come from the far circumcentres of nearly flat tets lying on a
// finely split oblique facet; a region of 100k+ tets costs one block seconds.
static void run_huge_regions(gq_ctx* c, const std::vector<int>& big) {
  int nb = (int)big.size();
  std::vector<int> st(nb);
  CK(cudaMemcpyAsync(c->tmpC, big.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, c->st));
  LAUNCH(k_status_of, nb, c->C, c->tmpC, nb, c->tmpA);
  d2h(c, st.data(), c->tmpA, 4 * (size_t)nb);
  std::vector<int> huge;
  for (int k = 0; k < nb; ++k) if (st[k] == CS_OVF) huge.push_back(big[k]);
  int nh = (int)huge.size();
  if (nh == 0) return;
  for (int mcap = std::max(c->C.ht, 16384);; mcap *= 2) {
    ensure_huge(c, nh, mcap);
    CK(cudaMemcpyAsync(c->hlist, huge.data(), 4 * (size_t)nh, cudaMemcpyHostToDevice, c->st));
    region_begin(c);
    k_region_huge<<<std::min(nh, c->HA.nblocks), BR_THREADS, 0, c->st>>>(c->D, c->C, c->SB, c->HA, c->hlist, nh);
    c->launches++;
    CK(cudaGetLastError());
    region_end(c);
    LAUNCH(k_status_of, nh, c->C, c->hlist, nh, c->tmpA);
    std::vector<int> hs(nh);
    d2h(c, hs.data(), c->tmpA, 4 * (size_t)nh);
    int still = 0;
    for (int k = 0; k < nh; ++k) still += hs[k] == CS_OVF;
    if (g_trace || c->verbose) std::fprintf(stderr, "[huge] %d cavities, capacity %d tets, %d overflow\n", nh, mcap, still);
    if (still == 0) return;
    if (mcap >= (1 << 16)) {   // beyond 64k tets: failed candidates (the sequential fallback skips them)
      LAUNCH(k_mark_memb, nh, c->C, c->hlist, nh, CS_OVF, MEMB_HUGE_OVF);   // the fallback skips them outright
      LAUNCH(k_set_status, nh, c->C, c->hlist, nh, CS_OVF, CS_CNSS);
      return;
    }
  }
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
  if (!o_thread_regions) {   // debug switch: per-thread kernel
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
    pull(c);
    unsigned long long rc = c->hc.region_calls, tested = c->hc.tested;
    float ms = 0; cudaEventElapsedTime(&ms, c->er0, c->er1);
    std::fprintf(stderr, "[region] launch %lld cands %d bytes_alg %llu ms %.3f\n", launch_no++, n1 - n0,
                 58ull * (tested - t_last) + 24ull * (rc - r_last), ms);
    t_last = tested; r_last = rc;
  }
  fine(c, 24);
  // overflow passes: the large warp tier, then one block per cavity
  ensure_tmp(c, n1 + 1);
  std::vector<int> hs(n1 - n0);
  stage(c, hs.data(), c->C.status + n0, sizeof(int) * (n1 - n0));
  sync(c);
  std::vector<int> ovf;
  for (int k = 0; k < n1 - n0; ++k) if (hs[k] == CS_OVF) ovf.push_back(n0 + k);
  std::vector<int> big;
  if (!ovf.empty() && WT1_MAXT != WT2_MAXT && !o_thread_regions) {
    int no = (int)ovf.size();
    CK(cudaMemcpyAsync(c->tmpB, ovf.data(), sizeof(int) * no, cudaMemcpyHostToDevice, c->st));
    region_begin(c);
    launch_warp_regions(c, k_region_warp<WT2_MAXT, WT2_HASH, 1>, WR_WARPS * sizeof(WarpShared2), no, 0, no, c->tmpB);
    region_end(c);
    LAUNCH(k_gather_status, no, c->C, c->tmpB, no, c->tmpA);
    stage(c, hs.data(), c->tmpA, sizeof(int) * no);
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
    run_huge_regions(c, big);
    sync(c);
    if (c->verbose && now_s() - tb > 0.5) std::fprintf(stderr, "[big] %d oversized cavities took %.2f s\n", nb, now_s() - tb);
    if (g_trace) {
      std::vector<int> nts(nb);
      int mx = 0; long long sm = 0;
      for (int k = 0; k < nb; ++k) {
        d2h(c, &nts[k], c->C.ntet + big[k], 4);
        mx = std::max(mx, nts[k]); sm += nts[k];
      }
      std::fprintf(stderr, "[big] n %d of %d tets max %d mean %.0f block %.3f ms\n", nb, n1 - n0, mx, (double)sm / nb, 1e3 * (now_s() - tb));
    }
  }
  fine(c, 26);
}

// rounds with at most this many candidates run the filter as one block
#ifndef SMALL_FILTER
#define SMALL_FILTER 64
#endif

// Contexts alive on each device.  A cooperative launch needs all its blocks
// resident at once; with several contexts running concurrently (C5) each one
// sizes its grid to its share of the device, so the cooperative grids of all
// of them fit together (their loops are grid-stride, any size is correct).
static std::atomic<int> g_ctx_count[64];
static int coop_share(gq_ctx* c, int full) {
  int k = std::max(1, g_ctx_count[c->device & 63].load());
  return std::max(1, full / k);
}

// candidates sorted by priority (class rank, hash, canonical tuple); smaller
// first (refine.py:45-52).  Two radix passes order by (class, hash); a run of
// equal (class, hash) -- a 64-bit splitmix collision -- is then put in
// canonical-tuple order by the thread at its head (growblast.py:49 compares
// the whole priority tuple).
__global__ void k_rank_keys(const __grid_constant__ Cand C, int n, unsigned long long* kh, unsigned int* kk, int* idx) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    bool ok = C.status[c] == CS_OK;
    kh[c] = ok ? C.h[c] : ~0ull;
    kk[c] = ok ? (unsigned int)C.kind[c] : 7u;
    idx[c] = c;
  }
}
__device__ __forceinline__ bool canon_less(int4 a, int4 b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  if (a.z != b.z) return a.z < b.z;
  return a.w < b.w;
}
__global__ void k_rank_ties(const __grid_constant__ Cand C, int* order, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += gridDim.x * blockDim.x) {
    int a = order[i];
    if (C.status[a] != CS_OK) continue;
    auto same = [&](int x, int y) { return C.status[y] == CS_OK && C.kind[x] == C.kind[y] && C.h[x] == C.h[y]; };
    if (i > 0 && same(order[i - 1], a)) continue;      // not the head of a run
    int j = i + 1;
    while (j < n && same(a, order[j])) ++j;
    for (int x = i + 1; x < j; ++x) {                  // insertion sort of the run by canon
      int v = order[x], y = x - 1;
      int4 cv = C.canon[v];
      while (y >= i && canon_less(cv, C.canon[order[y]])) { order[y + 1] = order[y]; --y; }
      order[y + 1] = v;
    }
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
  LAUNCH(k_rank_ties, n, c->C, c->tmpA, n);
  LAUNCH(k_rank_scatter, n, c->C, c->tmpA, n);
}

// LFMIS filter over candidates [0,n): state 0 for ok ones, 3 for the rest.
static void run_filter(gq_ctx* c, int n, int* nacc_out) {
  if (n <= 0) return;
  if (!o_filter_launches) {
    static int blocks_per_sm = 0, nsm = 0;
    if (!blocks_per_sm) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_filter_coop<false>, 256, 0));
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      if (blocks_per_sm < 1) throw std::runtime_error("filter kernel cannot be resident");
    }
    int blocks = std::min(coop_share(c, blocks_per_sm * nsm), (n + 7) / 8);
    int* ctr = c->d_int + 48;
    CK(cudaMemsetAsync(ctr, 0, 12, c->st));
    if (n <= SMALL_FILTER) {   // one block, no cooperative launch (same iterations, same result)
      k_filter_coop<true><<<1, 256, 0, c->st>>>(c->D, c->C, c->W, n, ctr);
      CK(cudaGetLastError());
    } else {
      void* args[] = {&c->D, &c->C, &c->W, &n, &ctr};
      CK(cudaLaunchCooperativeKernel((void*)k_filter_coop<false>, dim3(std::max(blocks, 1)), dim3(256), args, 0, c->st));
    }
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
  stage(c, h, c->d_int, 32);
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
  if (!c->tvn2) {
    c->tvn2 = dmalloc<int4>(2 * (size_t)D.tcap);
    c->sub2 = dmalloc<uint8_t>(D.tcap); c->seg2 = dmalloc<uint8_t>(D.tcap);
    c->ratio2 = dmalloc<double>(D.tcap); c->skip2 = dmalloc<uint8_t>(D.tcap);
  }
  TetRow tv2{c->tvn2}, tn2{c->tvn2 + 1};
  LAUNCH(k_compact_move, nt, D, c->tmpB, nt, tv2, tn2, c->sub2, c->seg2, c->ratio2, c->skip2);
  LAUNCH(k_compact_vt, c->hc.nv, D, c->tmpB, c->tmpA, c->hc.nv);
  c->tvn2 = D.tv.p; D.tv = tv2; D.tn = tn2;
  std::swap(D.sub, c->sub2); std::swap(D.seg, c->seg2);
  std::swap(D.ratio, c->ratio2); std::swap(D.skip, c->skip2);
  CK(cudaMemsetAsync(D.alive, 0, nt, c->st));
  CK(cudaMemsetAsync(D.alive, 1, na, c->st));
  CK(cudaMemsetAsync(&c->dctr->first_real, 0, sizeof(int), c->st));   // ids renumbered
  c->hc.nt = na;
  push(c);
}

static void ensure_big(gq_ctx* c, int need);
static void init_delaunay(gq_ctx* c, const int* order, int n) {
  CK(cudaMemcpyAsync(c->d_order, order, 4 * (size_t)n, cudaMemcpyHostToDevice, c->st));
  LAUNCH(k_init_first, 1, c->D, c->d_order, n, c->d_int + 8);
  sync(c);
  int first[4];
  d2h(c, first, c->d_int + 8, 16);
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
    d2h(c, P.data(), c->D.P, 24 * (size_t)n);
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
  double wf = getenv("GQ_INIT_WINDOW") ? atof(getenv("GQ_INIT_WINDOW")) : 0.03125;   // C2 sweep: 1/64 150, 1/32 132, 1/16 143, 1/8 167 ms
  fine(c, -1);
  int novf_last = 0;
  for (int round = 0; left > 0; ++round) {
    int W = (int)std::min<double>(left, std::max(64.0, wf * inserted));
    fine(c, 22);
    region_begin(c);
    if (!o_thread_init) {
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
    // big cavities (early rounds): resolve the lowest-order ones, truncate the window at the rest.
    // Only after a round that reported overflowed points in its window: otherwise the
    // cooperative filter below cuts the window at the first new one on the device, and
    // the block kernel picks it up next round -- no read-back here in the common case.
    std::vector<int> bl;
    if (novf_last > 0 || g_trace || o_init_launches) {
      CK(cudaMemsetAsync(c->d_int + 40, 0, 8, c->st));
      LAUNCH(k_count_ovf, W, C, d_plist, W, c->d_int + 40);
      int novf = read_int(c, c->d_int + 40);
      if (novf > 0) {
        std::vector<int> pl(W), sw(W);
        LAUNCH(k_gather_status, W, C, d_plist, W, d_scan);
        stage(c, pl.data(), d_plist, 4 * (size_t)W);
        stage(c, sw.data(), d_scan, 4 * (size_t)W);
        sync(c);
        for (int w = 0; w < W; ++w) if (sw[w] == CS_OVF) bl.push_back(pl[w]);
        if (WT1_MAXT != WT2_MAXT && !o_thread_init) {   // the large warp tier first
          int no = (int)bl.size();
          CK(cudaMemcpyAsync(d_keep, bl.data(), 4 * (size_t)no, cudaMemcpyHostToDevice, c->st));
          int blocks = std::min((no + WR_WARPS - 1) / WR_WARPS, c->S.nthreads / WR_WARPS);
          k_init_region_warp<WT2_MAXT, WT2_HASH, 1><<<std::max(blocks, 1), 32 * WR_WARPS, WR_WARPS * sizeof(WarpShared2), c->st>>>(
              c->D, C, c->S, d_pend, d_keep, no, d_hint, d_succ, d_touched, round, H, 1);
          c->launches++;
          CK(cudaGetLastError());
          LAUNCH(k_gather_status, no, C, d_keep, no, d_scan);
          std::vector<int> s2(no);
          stage(c, s2.data(), d_scan, 4 * (size_t)no);
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
        stage(c, sw.data(), d_scan, 4 * (size_t)W);
        sync(c);
        for (int w = 0; w < W; ++w) if (sw[w] == CS_OVF) { W = w; break; }
        if (W == 0) throw std::runtime_error("init: cavity overflow");
        CK(cudaMemcpyAsync(c->tmpC, bl.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, c->st));
        }
      }
    }
    fine(c, 1);
    int nacc = 0, add_t = 0;
    if (!o_init_launches) {
      static int bps = 0, nsm = 0;
      if (!bps) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_init_filter_coop<false>, 256, 0));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        if (bps < 1) throw std::runtime_error("init filter kernel cannot be resident");
      }
      int blocks = std::max(1, std::min(coop_share(c, bps * nsm), (W + 7) / 8));
      int* tot = c->d_int + 52;
      if (W <= SMALL_FILTER) {
        k_init_filter_coop<true><<<1, 256, 0, c->st>>>(c->D, C, c->W, d_plist, W, nt, d_acc, d_plist2, d_scan, tot, d_succ);
        CK(cudaGetLastError());
      } else {
        void* args[] = {&c->D, &C, &c->W, &d_plist, &W, &nt, &d_acc, &d_plist2, &d_scan, &tot, &d_succ};
        CK(cudaLaunchCooperativeKernel((void*)k_init_filter_coop<false>, dim3(blocks), dim3(256), args, 0, c->st));
      }
      c->launches++;
      int h2[4];
      stage(c, h2, tot, 16);
      sync(c);
      nacc = h2[0]; add_t = h2[1]; novf_last = h2[2];
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
      stage(c, &lastn, d_keep + W - 1, 4);
      stage(c, &lasts, d_scan + W - 1, 4);
      exclusive_scan(c, d_acc, d_plist2, W);
      int lastacc_scan = 0;
      stage(c, &lastacc_scan, d_plist2 + W - 1, 4);
      stage(c, &lasta, d_acc + W - 1, 4);
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
      pull(c); unsigned long long rc = c->hc.region_calls;
      static unsigned long long rc_last = 0;
      std::fprintf(stderr, "[init] round %d W %d big %d acc %d nt %d region_ms %.3f computed %llu maxtet %d\n", round, W,
                   (int)bl.size(), nacc, nt, rms, rc - rc_last, read_int(c, c->d_int + 41));
      rc_last = rc;
    }
    left -= nacc;
    inserted += nacc;
    c->hc.nt = nt;
    push(c);
    if (nacc == 0 && novf_last == 0) throw std::runtime_error("init made no progress");
    c->init_rounds = round + 1;
    fine(c, 6);
  }
  // big-slab candidates must not keep stale bigi for the refinement rounds
  sync(c);
  dfree(d_pend); dfree(d_hint); dfree(d_plist); dfree(d_plist2); dfree(d_acc);
  dfree(d_scan); dfree(d_keep); dfree(d_succ); dfree(d_touched); dfree(H.cellv);
}

// ------------------------------------------------------------------ round

__global__ void k_states(const __grid_constant__ Dev D, const __grid_constant__ Cand C, int n, int* okf, int* failf) {
  unsigned long long claims = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    int st = C.status[c];
    int s = st == CS_OK ? 0 : (st == CS_DROP ? -1 : 3);
    C.state[c] = s;
    okf[c] = s == 0;
    failf[c] = s == 3;
    if (s == 0) claims += C.ntet[c] + C.nbf[c] + C.ncr[c] + C.nbseg[c] + C.neseg[c] + (C.extra[c] >= 0);
  }
  if (claims) atomicAdd(&D.ctr->claims, claims);
}
__global__ void k_kept(const __grid_constant__ Cand C, int n, int* keep) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) keep[c] = C.status[c] != CS_DROP;
}
__global__ void k_acc_byrank(const __grid_constant__ Cand C, int n, int* byrank) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    if (C.state[c] == 1) byrank[C.rank[c]] = c;
}
__global__ void k_nonneg(const int* a, int n, int* f) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) f[i] = a[i] >= 0;
}
__global__ void k_gather_i32(const int* src, const int* idx, int n, int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}
__global__ void k_item_count(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* ins, int ni, int* cnt) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ni; k += gridDim.x * blockDim.x) {
    int c = ins[k], kind = C.kind[c];
    if (kind == K_SEG) { int sid = D.sg_sid[C.tgt[c]]; cnt[k] = D.segpoly_off[sid + 1] - D.segpoly_off[sid]; }
    else cnt[k] = kind == K_FACE ? 1 : 0;
  }
}
__global__ void k_item_fill(const __grid_constant__ Dev D, const __grid_constant__ Cand C, const int* ins, int ni, const int* off, const int* cnt, T2Items T, int* item_of) {
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
__global__ void k_count_seed_dead(const __grid_constant__ Dev D, const __grid_constant__ Cand C, int n, int* out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (C.state[c] != 2 || C.kind[c] != K_TET) continue;
    atomicAdd(out, 1);
    if (!D.alive[C.tgt[c]]) atomicAdd(out + 1, 1);
  }
}
__global__ void k_bump(const __grid_constant__ Dev D, int dnv, int dnt) { D.ctr->nv += dnv; D.ctr->nt += dnt; }
__global__ void k_pool_pos(const __grid_constant__ Cand C, int n, const int* keepscan, const int* keep) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    C.pool[c] = keep[c] ? keepscan[c] : -1;
}

struct RoundOut {
  int phase = -1; long long ncand = 0, acc = 0, rej = 0, failed = 0, inserted = 0;
  double vt[6] = {0, 0, 0, 0, 0, 0};   // verbose only: pool+regions, filter, insert, fallback, post (synchronised)
  int st_hist[6] = {0, 0, 0, 0, 0, 0}; // verbose only: candidate status histogram (CS_*)
  int waves = 0;                       // fallback waves
};
// verbose diagnostics: stage boundary with a stream sync (never on the timed path)
static double vmark(gq_ctx* c, double& last) {
  CK(cudaStreamSynchronize(c->st));
  double t = now_s(), d = t - last;
  last = t;
  return d;
}


static const char* g_prof_names[8] = {"pool", "regions", "filter", "insert", "2d", "fallback", "post", "other"};

// scan of n ints; returns the total
static int scan_total(gq_ctx* c, const int* in, int* out, int n) {
  if (n <= 0) return 0;
  exclusive_scan(c, in, out, n);
  int a = 0, b = 0;
  stage(c, &a, in + n - 1, 4);
  stage(c, &b, out + n - 1, 4);
  sync(c);
  return a + b;
}

#include "gq_grow.cuh"

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
  {
    int blocks = std::max(1, std::min((na + WS_WARPS - 1) / WS_WARPS, c->SB.nthreads / WS_WARPS));
    k_star_check<<<blocks, 32 * WS_WARPS, WS_WARPS * sizeof(StarShared), c->st>>>(c->D, C, acc, na, flags, c->SB, c->L, round_no);
    c->launches++;
    CK(cudaGetLastError());
  }
  int ni = select_flagged(c, flags, na, pos);
  *inserted += ni;
  if (ni == 0) return;
  LAUNCH(k_gather_i32, ni, acc, pos, ni, ins);
  pull(c);
  int nv = c->hc.nv, nt = c->hc.nt;
  LAUNCH(k_gather_nbf, ni, C, ins, ni, flags);
  int tot = scan_total(c, flags, pos, ni);
  ensure_mesh_room(c, (long long)nv + ni, (long long)nt + tot);
  ensure_round_room(c, ni, c->npoly > 0 ? 8LL * ni : 0);
  LAUNCH(k_assign_ids, ni, C, ins, ni, pos, nv, nt);
  Ins I; I.list = ins; I.n = ni; I.nv0 = nv; I.nt0base = nt;
  fine(c, 18);
  LAUNCH(k_ins_vertices, ni, c->D, C, I);
  fine(c, 32);
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
  fine(c, 33);
  double t1 = now_s();
  static const int t2_fused_max = getenv("GQ_T2_FUSED_MAX") ? atoi(getenv("GQ_T2_FUSED_MAX")) : 256;
  static const bool t2_thread = getenv("GQ_T2_THREAD") != nullptr;
  if (nit > 0 && nit <= t2_fused_max) {   // few items: all passes in one launch, polygons split over blocks
    c->T.n = nit;
    CK(cudaMemsetAsync(c->d_int + 16, 0, 4, c->st));
    if (t2_thread) k_t2_fused<false><<<std::min(std::min(nit, c->npoly), c->S.nthreads / 128), 128, 0, c->st>>>(c->D, C, c->T, c->S, c->d_int + 16);
    else k_t2_fused<true><<<std::min(std::min(nit, c->npoly), c->S.nthreads / 8), 256, 0, c->st>>>(c->D, C, c->T, c->S, c->d_int + 16);
    c->launches++;
    CK(cudaGetLastError());
  } else if (nit > 0) {
    c->T.n = nit;
    int left = nit;
    for (int pass = 0; left > 0; ++pass) {
      CK(cudaMemsetAsync(c->d_int + 16, 0, 4, c->st));
      if (t2_thread) {
        LAUNCH_S(k_t2_compute, nit, c->D, C, c->T, c->S);
        LAUNCH(k_t2_claim, nit, c->D, C, c->T);
        LAUNCH_S(k_t2_apply, nit, c->D, C, c->T, c->S, c->d_int + 16);
        LAUNCH(k_t2_reset, nit, c->D, C, c->T, 1);
        LAUNCH_S(k_t2_commit, nit, c->D, C, c->T, c->S);
      } else {
        LAUNCH_W(k_t2w_compute, nit, c->D, C, c->T, c->S);
        LAUNCH_W(k_t2w_claim, nit, c->D, C, c->T);
        LAUNCH_W(k_t2w_apply, nit, c->D, C, c->T, c->d_int + 16);
        LAUNCH_W(k_t2w_reset, nit, c->D, c->T, 1);
        LAUNCH_W(k_t2w_commit, nit, c->D, C, c->T, c->S);
      }
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
  fine(c, 34);
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

// GQ_WATCHDOG=<seconds>: a thread reports the host driver's current stage and
// round whenever it has not moved for that long (locating device stalls)
static std::atomic<int> g_wd_stage{-2}, g_wd_round{-1};
static std::atomic<long long> g_wd_tick{0};
static void watchdog_start() {
  static std::once_flag once;
  const char* e = getenv("GQ_WATCHDOG");
  if (!e) return;
  double secs = atof(e);
  std::call_once(once, [secs] {
    std::thread([secs] {
      long long last = -1; double since = now_s();
      for (;;) {
        std::this_thread::sleep_for(std::chrono::milliseconds(500));
        long long t = g_wd_tick.load();
        if (t != last) { last = t; since = now_s(); continue; }
        if (now_s() - since > secs) {
          std::fprintf(stderr, "[watchdog] no progress for %.0f s: round %d stage %d\n", now_s() - since,
                       g_wd_round.load(), g_wd_stage.load());
          since = now_s();
        }
      }
    }).detach();
  });
}
static void fine(gq_ctx* c, int k) {
  g_wd_stage.store(k); g_wd_tick.fetch_add(1);
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
  double vlast = c->verbose ? now_s() : 0;
  c->big_used = 0;
  if (o_trace_from >= 0) g_trace = round_no >= o_trace_from;   // stage trace from a round on
  g_wd_round.store(round_no);
  pull(c);
  maintain_capacity(c);
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
    if (g_grid_thread) LAUNCH(k_grid_cands, nbase, c->D, c->G, c->C, 0, nbase);
    else LAUNCH_W(k_grid_cands_w, nbase, c->D, c->G, c->C, 0, nbase);
    fine(c, 28);
    CK(cudaMemsetAsync(c->d_int + 60, 0, 8, c->st));
    LAUNCH(k_redirect, nbase, c->D, c->C, 0, nbase, c->d_int + 60);
    fine(c, 13);
    ensure_tmp(c, nbase + 1);
    LAUNCH(k_kept, nbase, c->C, nbase, c->Q.a);
    int redir[2] = {0, 0};
    stage(c, redir, c->d_int + 60, 8);   // read with the scan below
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
  if (c->verbose) {
    R.vt[0] = vmark(c, vlast);
    std::vector<int> st(n);
    if (n) d2h(c, st.data(), c->C.status, 4 * (size_t)n);
    for (int v : st) if (v >= 0 && v < 6) R.st_hist[v]++;
    vlast = now_s();
  }
  double t1 = now_s();
  ensure_tmp(c, n + 1);
  LAUNCH(k_states, n, c->D, c->C, n, c->Q.a, c->Q.b);
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
  if (c->verbose) R.vt[1] = vmark(c, vlast);
  insert_accepted(c, n, &R.acc, &R.inserted, round_no);
  if (c->verbose) R.vt[2] = vmark(c, vlast);
  R.rej = nok - R.acc;
  t1 = now_s();
  fine(c, -1);
  if (nfail > 0) {
    pull(c);
    ensure_mesh_room(c, (long long)c->hc.nv + nfail, (long long)c->hc.nt + 1024LL * nfail + 65536);
    ensure_round_room(c, nfail, c->npoly > 0 ? 8LL * nfail : 0);
    FallbackIO F; F.list = c->Q.h; F.n = nfail; F.round_no = round_no; F.seed = c->seed;
    F.with_facets = c->npoly > 0; F.lmin2 = lmin2; F.inserted = c->d_int + 20;
    CK(cudaMemsetAsync(c->d_int + 20, 0, 4, c->st));
    if (o_fallback_serial) {
      k_fallback<<<1, 1, 0, c->st>>>(c->D, c->C, c->SB, F, c->T, c->L);
      c->launches++;
      CK(cudaGetLastError());
    } else {
      // waves (gq_fallback.cuh): parallel evaluation, in-order application
      int* out = dmalloc<int>(2 * (size_t)nfail);
      F.window = o_fb_window;
      int h0[2] = {0, std::min(nfail, F.window)};
      CK(cudaMemcpyAsync(c->d_int + 24, h0, 8, cudaMemcpyHostToDevice, c->st));
      int start = 0, waves = 0;
      while (start < nfail) {
        LAUNCH_S(k_fb_scan, std::min(nfail - start, F.window), c->D, c->C, c->S, F, c->T, c->L, c->d_int + 24, out, c->d_int + 25);
        k_fb_apply<<<1, 1, 0, c->st>>>(c->D, c->C, c->SB, F, c->T, c->L, c->d_int + 24, out, c->d_int + 25);
        c->launches++;
        CK(cudaGetLastError());
        start = read_int(c, c->d_int + 24);
        ++waves;
      }
      dfree(out);
      R.waves = waves;
      if (g_trace) std::fprintf(stderr, "[fallback] round %d: %d candidates in %d waves\n", round_no, nfail, waves);
    }
    R.inserted += read_int(c, c->d_int + 20);
  }
  fine(c, 30);
  if (c->verbose) R.vt[3] = vmark(c, vlast);
  if (g_trace && phase == 2) {   // how many blasted tet candidates had their own tet taken by an accepted cavity
    CK(cudaMemsetAsync(c->d_int + 56, 0, 8, c->st));
    LAUNCH(k_count_seed_dead, n, c->D, c->C, n, c->d_int + 56);
    int h2[2];
    d2h(c, h2, c->d_int + 56, 8);
    std::fprintf(stderr, "[seed] round %d rejected %d with dead seed tet %d\n", round_no, h2[0], h2[1]);
  }
  g_prof[5] += now_s() - t1;
  t1 = now_s();
  // post round: new vertices vs every constraint ball, then new / dirty
  // constraints vs the vertices around them
  fine(c, -1);
  grid_sync(c);
  fine(c, 7);
  if (c->hc.nv > c->reg_nv) {
    if (g_grid_thread) LAUNCH(k_grid_newverts, c->hc.nv - c->reg_nv, c->D, c->G, c->reg_nv, c->hc.nv);
    else LAUNCH_W(k_grid_newverts_w, c->hc.nv - c->reg_nv, c->D, c->G, c->reg_nv, c->hc.nv);
  }
  c->reg_nv = c->hc.nv;
  fine(c, 8);
  CK(cudaMemsetAsync(c->d_int, 0, 16, c->st));
  CK(cudaMemsetAsync(&c->dctr->chk, 0, sizeof(c->dctr->chk), c->st));
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
  if (c->verbose) R.vt[4] = vmark(c, vlast);
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
  watchdog_start();
  { int ws = getenv("GQ_WSTOP") ? atoi(getenv("GQ_WSTOP")) : 0; CK(cudaMemcpyToSymbolAsync(g_wstop, &ws, 4, 0, cudaMemcpyHostToDevice, c->st)); }
  c->n_input = n_input; c->npoly = f;
  c->rounds.clear(); c->rtimes.clear(); c->launches = 0; c->region_ms = 0;
  free_all(c);
  err_baseline(c);   // (g_err / g_errn are never reset: other contexts may be running)
  unsigned long long z4[4] = {0, 0, 0, 0};
  CK(cudaMemcpyToSymbolAsync(g_exact_calls, z4, 32, 0, cudaMemcpyHostToDevice, c->st));
  int npidx = f > 0 ? poff[f] : 0;
  double ta = now_s();
  alloc_mesh(c, n, m, f, npidx);
  CK(cudaStreamSynchronize(c->st));
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
  CK(cudaMemsetAsync(c->dctr, 0, sizeof(Counters), c->st));
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
    CK(cudaMemcpyAsync(D.poly_keep, keep, 8 * (size_t)f, cudaMemcpyHostToDevice, c->st));
    std::vector<uint8_t> obl(f, 1);
    for (int pid = 0; pid < f; ++pid)
      for (int k = 0; k < 3 && obl[pid]; ++k) {
        bool same = true;
        for (int q = poff[pid] + 1; q < poff[pid + 1] && same; ++q) same = xyz[3 * pidx[q] + k] == xyz[3 * pidx[poff[pid]] + k];
        if (same) obl[pid] = 0;
      }
    CK(cudaMemcpyAsync(D.poly_obl, obl.data(), f, cudaMemcpyHostToDevice, c->st));
    D.poly_obl_hull = 0;   // the hull guards act only where a ghost tet touches the split element
    for (int pid = 0; pid < f && !D.poly_obl_hull; ++pid) D.poly_obl_hull = obl[pid];
    if (!sp.empty()) CK(cudaMemcpyAsync(D.segpoly, sp.data(), 4 * sp.size(), cudaMemcpyHostToDevice, c->st));
  }
  CK(cudaMemcpyAsync(D.segpoly_off, spo.data(), 4 * (size_t)(m + 1), cudaMemcpyHostToDevice, c->st));
  // small-angle apexes: input vertices where two input segments meet at < 45
  // degrees get concentric-shell splitting (seg_split_point, gq_cand.cuh)
  {
    std::vector<uint8_t> apex(std::max(n, 1), 0);
    std::vector<int> deg(n + 1, 0), adj(2 * (size_t)m);
    for (int s = 0; s < m; ++s) { deg[seg[2 * s] + 1]++; deg[seg[2 * s + 1] + 1]++; }
    for (int v = 0; v < n; ++v) deg[v + 1] += deg[v];
    std::vector<int> fill(deg.begin(), deg.end() - 1);
    for (int s = 0; s < m; ++s) { adj[fill[seg[2 * s]]++] = seg[2 * s + 1]; adj[fill[seg[2 * s + 1]]++] = seg[2 * s]; }
    const double c45 = std::sqrt(0.5);
    for (int v = 0; v < n; ++v) {
      for (int i = deg[v]; i < deg[v + 1] && !apex[v]; ++i) {
        const double* a = xyz + 3 * (size_t)v;
        const double* x = xyz + 3 * (size_t)adj[i];
        double u0[3] = {x[0] - a[0], x[1] - a[1], x[2] - a[2]};
        double lu = std::sqrt(u0[0] * u0[0] + u0[1] * u0[1] + u0[2] * u0[2]);
        for (int j = i + 1; j < deg[v + 1]; ++j) {
          const double* y = xyz + 3 * (size_t)adj[j];
          double w0[3] = {y[0] - a[0], y[1] - a[1], y[2] - a[2]};
          double lw = std::sqrt(w0[0] * w0[0] + w0[1] * w0[1] + w0[2] * w0[2]);
          if (u0[0] * w0[0] + u0[1] * w0[1] + u0[2] * w0[2] > c45 * lu * lw) { apex[v] = 1; break; }
        }
      }
    }
    D.vapex = dmalloc<uint8_t>(std::max(n, 1));
    CK(cudaMemcpyAsync(D.vapex, apex.data(), std::max(n, 1), cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  // init_delaunay
  init_delaunay(c, order, n);
  CK(cudaEventRecord(c->ev1, c->st));
  sync(c);
  float ims = 0; cudaEventElapsedTime(&ims, c->ev0, c->ev1); c->init_ms = ims;
  // constraints
  if (m > 0) {
    int* dseg = dmalloc<int>(2 * (size_t)m);
    CK(cudaMemcpyAsync(dseg, seg, 8 * (size_t)m, cudaMemcpyHostToDevice, c->st));
    LAUNCH(k_segs_init, m, D, dseg, m);
    sync(c);
    dfree(dseg);
  }
  pull(c);
  c->hc.nsegrec = m;
  push(c);
  if (f > 0) {
    int* dpo = dmalloc<int>(f + 1); int* dpi = dmalloc<int>(std::max(npidx, 1));
    CK(cudaMemcpyAsync(dpo, poff, 4 * (size_t)(f + 1), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(dpi, pidx, 4 * (size_t)npidx, cudaMemcpyHostToDevice, c->st));
    D.poly_off = dpo; D.poly_idx = dpi;        // resident: non-convex polygons' inside test
    LAUNCH(k_poly_convex, f, D, f);
    LAUNCH_S(k_facets_init, f, D, dpo, dpi, f, c->S, (int*)nullptr);
    sync(c);
    pull(c);
    LAUNCH(k_facets_records, c->hc.nt2, D, c->hc.nt2);
    sync(c);
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
    d2h(c, h, c->d_int + 4, 16);
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    c->rounds.push_back({round_no, R.phase, R.ncand, R.acc, R.rej, R.failed, R.inserted, h[2], h[3]});
    c->rtimes.push_back(dt);
    if (c->verbose) {
      pull(c);
      const unsigned int* k = c->hc.chk;
      std::fprintf(stderr, "round %d phase=%d candidates=%lld accepted=%lld blasted=%lld failed=%lld inserted=%lld time=%.4f"
                   " | nv %d nt %d segs %d faces %d skipped %d | check: seg miss %u enc %u (collinear %u) face miss %u enc %u (coplanar %u)"
                   " | skips seg %u/%u/%u/%u face %u/%u/%u/%u tet %u/%u/%u/%u | fails %u/%u/%u/%u/%u/%u/%u/%u\n",
                   round_no, R.phase, R.ncand, R.acc, R.rej, R.failed, R.inserted, dt, c->hc.nv, c->hc.nt, c->hc.nsegrec,
                   c->hc.nfacerec, c->hc.nskip, k[0], k[1], k[2], k[3], k[4], k[5], c->hc.skipr[0], c->hc.skipr[1],
                   c->hc.skipr[2], c->hc.skipr[3], c->hc.skipr[4], c->hc.skipr[5], c->hc.skipr[6], c->hc.skipr[7],
                   c->hc.skipr[8], c->hc.skipr[9], c->hc.skipr[10], c->hc.skipr[11], c->hc.fail[0], c->hc.fail[1],
                   c->hc.fail[2], c->hc.fail[3], c->hc.fail[4], c->hc.fail[5], c->hc.fail[6], c->hc.fail[7]);
      std::fprintf(stderr, "  stages ms: pool+regions %.1f filter %.1f insert %.1f fallback %.1f post %.1f"
                   " | status ok %d cnss %d tooclose %d memb %d ovf %d drop %d | fallback waves %d, slowest eval %.2f ms (outcome %d kind %d)\n",
                   1e3 * R.vt[0], 1e3 * R.vt[1], 1e3 * R.vt[2], 1e3 * R.vt[3], 1e3 * R.vt[4], R.st_hist[0],
                   R.st_hist[1], R.st_hist[2], R.st_hist[3], R.st_hist[4], R.st_hist[5], R.waves,
                   (double)(c->hc.fb_slow >> 8) / 1.965e6, (int)((c->hc.fb_slow >> 4) & 15), (int)(c->hc.fb_slow & 15));
      std::fprintf(stderr, "  star queries: stale starts %llu (tets scanned %llu), large-arena reruns %llu, lock spins %llu;"
                   " walks past the cap %llu (randomised steps ~%llu)\n",
                   c->hc.vq[0], c->hc.vq[1], c->hc.vq[2], c->hc.vq[3], c->hc.vq[4], c->hc.vq[5]);
      std::fprintf(stderr, "  slow fallback evaluations: %llu, Mcycles make %.1f hull walk %.1f seeds %.1f region %.1f\n",
                   c->hc.vq[10], c->hc.vq[6] / 1024.0, c->hc.vq[7] / 1024.0, c->hc.vq[8] / 1024.0, c->hc.vq[9] / 1024.0);
      c->hc.fb_slow = 0;
      CK(cudaMemsetAsync(&c->dctr->fb_slow, 0, 8, c->st));
    }
    round_no += 1;
  }
  CK(cudaEventRecord(c->ev1, c->st));
  sync(c);
  float ms = 0; cudaEventElapsedTime(&ms, c->ev0, c->ev1); c->dev_ms = ms;
  resolve_events(c);
  if (g_fine || g_fine_ev) {
    std::fprintf(stderr, "[gq fine]");
    for (int k = 0; k < 40; ++k) if (g_fine_t[k] > 0) { std::fprintf(stderr, " %s %.1f;", g_fine_names[k], 1000 * g_fine_t[k]); g_fine_t[k] = 0; }
    std::fprintf(stderr, "\n");
  }
  if (getenv("GQ_PROFILE")) {
    std::fprintf(stderr, "[gq profile] init %.1f ms (%d rounds);", c->init_ms, c->init_rounds);
    for (int k = 0; k < 8; ++k) { std::fprintf(stderr, " %s %.1f ms;", g_prof_names[k], 1000 * g_prof[k]); g_prof[k] = 0; }
    std::fprintf(stderr, " region kernels %.1f ms; launches %lld\n", c->region_ms, c->launches);
    pull(c);
    std::fprintf(stderr, "[gq 2d] cavities %llu walk steps %llu exhaustive scans %llu (%llu triangles)\n", c->hc.t2st[0],
                 c->hc.t2st[1], c->hc.t2st[2], c->hc.t2st[3]);
  }
  pull(c);
  if (out) {
    std::memset(out, 0, sizeof(*out));
    out->nv = c->hc.nv; out->nt = c->hc.nt;
    // live constraint counts
    std::vector<unsigned int> sf(c->hc.nsegrec), ff(c->hc.nfacerec);
    d2h(c, sf.data(), D.sg_fl, 4 * sf.size());
    d2h(c, ff.data(), D.sf_fl, 4 * ff.size());
    for (auto x : sf) out->n_subsegments += (x & RF_LIVE) ? 1 : 0;
    for (auto x : ff) out->n_subfaces += (x & RF_LIVE) ? 1 : 0;
    out->n_rounds = (int64_t)c->rounds.size();
    out->n_skipped = std::min(c->hc.nskip, c->L.cap);
    unsigned long long ex[4];
    CK(cudaMemcpyFromSymbol(ex, g_exact_calls, 32));
    for (int k = 0; k < 4; ++k) out->exact_calls[k] = (int64_t)ex[k];
    out->device_ms = c->dev_ms; out->init_ms = c->init_ms;
    out->kernel_launches = c->launches;
    unsigned long long rc = c->hc.region_calls, tested = c->hc.tested;
    out->region_calls = (int64_t)rc;
    out->region_ms = c->region_ms;
    std::vector<uint8_t> org2(c->hc.nv);
    d2h(c, org2.data(), D.vorigin, c->hc.nv);
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
    out->n_cand = (int64_t)c->hc.cands; out->t_tested = (int64_t)tested; out->k_claims = (int64_t)c->hc.claims;
    out->t_created = (int64_t)c->hc.created; out->t_deleted = (int64_t)c->hc.deleted;
    out->bytes_refine = 144 * out->n_cand + 58 * out->t_tested + 8 * out->k_claims + 51 * out->t_created +
                        out->t_deleted + 29 * (int64_t)(c->hc.nv - n);
  }
}

