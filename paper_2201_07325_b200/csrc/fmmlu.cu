// libfmmlu: C ABI + host orchestration of the RS-S factorization on one B200.
//
// Host C++ keeps only integer bookkeeping (tree, owners, index lists, task
// descriptors); every floating-point step of the method runs in the CUDA kernels
// of kernels.cu / gemm.cu:
//   level ℓ = L-1 … 2:
//     build the level's block-sparse current-matrix store ("BSR": one dense block
//       per owner pair at Chebyshev separation ≤ 2, entries = pure kernel or the
//       Schur-updated value carried over from level ℓ+1)          [k_build_level]
//     colour c = 0 … 7 (reading C8; boxes of one colour are independent):
//       M = [A_QB; A_BQᵀ; proxy rows]       [k_copy, k_proxy]
//       ID → perm, k; T = R11⁻¹R12 (Gram + pivoted Cholesky or
//       TSQR + CPQR, reading R4)                                    [DMMA GEMM, k_pchol_reg, k_trsm_T]
//       E/F transforms with T (Eq. pap … X blocks, L739-788)      [DMMA GEMM]
//       X_RR⁻¹ (Gauss-Jordan), Up = X_RR⁻¹X_{R(S∪N)}; X_{(S∪N)R} is kept in place of Lp   [k_gj_reg, GEMM]
//       Schur update Δ_{(S∪N)²} −= X_{(S∪N)R}·Up scattered into the BSR (L813-825) [GEMM+atomics]
//   root: B_t dense block → X⁻¹ (L894-918)                        [k_build, blocked GJ: k_gj_panel_reg + DMMA updates]
// Solve: upward sweep over phases, root apply, downward sweep.
#include <cuda_runtime.h>
#include <malloc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <condition_variable>
#include <functional>
#include <future>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "../../include/fmmlu.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "devtree.h"
#include "tree.h"

using namespace fmmlu;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// --------------------------------------------------------------------------- device memory
// host-side time spent in allocator calls (FMMLU_TRACE diagnostics)
struct AllocClock {
  double alloc_ms = 0, free_ms = 0, pin_ms = 0, alloc_max = 0;
  long long nalloc = 0;
};
AllocClock g_ac;
double wall_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Process-wide cache of large device blocks.  Repeated factorizations ask for the same large
// buffers (level block stores, workspaces); handing them back to cudaMallocAsync's pool and
// re-requesting them occasionally stalls the host for hundreds of ms (pool growth / reclaim),
// so blocks ≥ kBigBlock are kept here (allocated from, and evicted to, the async pool).  Reuse
// is stream-ordered: an event recorded at release is waited on by the next user's stream.  The
// cache holds at most kBigCap bytes (oldest blocks are evicted first); a failed allocation
// evicts everything and retries.
constexpr size_t kBigBlock = 32u << 20;
constexpr int kMaxDev = 64;

// The library's own stream-ordered pool per device (never the device's default pool, which other
// libraries in the process share): release threshold = max, so memory freed by one factorization is
// reused by the next without going back to the driver.  fmmlu_release_cache() trims it.
cudaMemPool_t lib_pool(int dev) {
  static std::mutex mu;
  static cudaMemPool_t pools[kMaxDev] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= kMaxDev) throw Error(FMMLU_ECUDA, "device ordinal out of range");
  if (!pools[dev]) {
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    FMMLU_CUDA(cudaMemPoolCreate(&pools[dev], &pp));
    uint64_t thr = UINT64_MAX;
    FMMLU_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return pools[dev];
}

int cur_dev() {
  int d = 0;
  FMMLU_CUDA(cudaGetDevice(&d));
  return d;
}

// Process-wide cache of large device blocks, one per device.  Repeated factorizations ask for the
// same large buffers (factor-store chunks, workspaces); handing them back to the pool and
// re-requesting them occasionally stalls the host for hundreds of ms (pool growth / reclaim), so
// blocks ≥ kBigBlock are kept here (allocated from, and evicted to, the library pool).  Reuse is
// stream-ordered: an event recorded at release is waited on by the next user's stream.  The cache
// holds at most `cap` bytes (oldest blocks are evicted first); a failed allocation evicts
// everything and retries; fmmlu_release_cache() empties it.
struct BigCache {
  struct Blk {
    void* p;
    size_t bytes;
    cudaEvent_t ev;
  };
  int dev = 0;
  size_t cap = 0;  // FMMLU_CACHE_PCT (default 60) % of device memory (set on first use)
  std::mutex mu;
  std::vector<Blk> free_;  // oldest first
  size_t held = 0;
  void* take(size_t b, cudaStream_t st, size_t* got) {
    std::lock_guard<std::mutex> lk(mu);
    int best = -1;
    for (int i = 0; i < (int)free_.size(); ++i)
      if (free_[i].bytes >= b && free_[i].bytes <= 2 * b + kBigBlock &&
          (best < 0 || free_[i].bytes < free_[best].bytes))
        best = i;
    if (best < 0) return nullptr;
    Blk k = free_[best];
    free_.erase(free_.begin() + best);
    held -= k.bytes;
    cudaStreamWaitEvent(st, k.ev, 0);
    cudaEventDestroy(k.ev);
    *got = k.bytes;
    return k.p;
  }
  // caller holds mu and has this cache's device current; st = a live stream of the caller (the
  // releasing stream may be gone), or null: free synchronously
  void evict_front(cudaStream_t st) {
    Blk k = free_.front();
    free_.erase(free_.begin());
    held -= k.bytes;
    if (st) {
      cudaStreamWaitEvent(st, k.ev, 0);
      cudaFreeAsync(k.p, st);
    } else {
      cudaEventSynchronize(k.ev);
      cudaFree(k.p);
    }
    cudaEventDestroy(k.ev);
  }
  void give(void* p, size_t bytes, cudaStream_t st) {
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, st) != cudaSuccess) {  // no ordering possible: free synchronously
      cudaGetLastError();
      cudaDeviceSynchronize();
      cudaFree(p);
      return;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (cap == 0) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      static const int pct = getenv("FMMLU_CACHE_PCT") ? atoi(getenv("FMMLU_CACHE_PCT")) : 60;
      cap = tot / 100 * (size_t)std::max(0, std::min(95, pct));
    }
    free_.push_back({p, bytes, ev});
    held += bytes;
    while (held > cap && free_.size() > 1) evict_front(st);
  }
  void flush(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(mu);
    while (!free_.empty()) evict_front(st);
  }
  size_t cached() {
    std::lock_guard<std::mutex> lk(mu);
    return held;
  }
};
// never destroyed (no CUDA calls from static destructors at process exit)
BigCache& big_cache(int dev) {
  static BigCache* c[kMaxDev] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= kMaxDev) throw Error(FMMLU_ECUDA, "device ordinal out of range");
  if (!c[dev]) {
    c[dev] = new BigCache();
    c[dev]->dev = dev;
  }
  return *c[dev];
}

// Last resort of a failed allocation: the pool keeps every freed byte reserved (release threshold
// = max), and after several factorizations with different block sizes that reservation is
// fragmented, so one large request can fail with enough memory idle.  Wait for the stream, hand the
// idle reservation back to the driver and retry once.
cudaError_t retry_trimmed(void** p, size_t bytes, cudaStream_t s) {
  cudaGetLastError();
  cudaStreamSynchronize(s);
  cudaMemPool_t pool = lib_pool(cur_dev());
  cudaMemPoolTrimTo(pool, 0);
  cudaError_t e = cudaMallocFromPoolAsync(p, bytes, pool, s);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept
      : p(o.p), bytes(o.bytes), st(o.st), big(o.big), borrowed(o.borrowed), cap(o.cap), dev(o.dev) {
    o.p = nullptr;
    o.bytes = 0;
    o.big = false;
    o.borrowed = false;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      st = o.st;
      big = o.big;
      borrowed = o.borrowed;
      cap = o.cap;
      dev = o.dev;
      o.p = nullptr;
      o.bytes = 0;
      o.big = false;
      o.borrowed = false;
    }
    return *this;
  }
  ~DBuf() { release(); }
  bool big = false;       // from / back to the big-block cache
  bool borrowed = false;  // points into a staging arena (released with the arena)
  void release() {
    if (borrowed) {
      p = nullptr;
      bytes = 0;
      borrowed = false;
      return;
    }
    if (p) {
      const double t0 = wall_ms();
      if (big) big_cache(dev).give(p, cap, st);
      else cudaFreeAsync(p, st);
      g_ac.free_ms += wall_ms() - t0;
    }
    p = nullptr;
    bytes = 0;
    big = false;
  }
  size_t cap = 0;
  int dev = 0;  // the device it lives on (the caller's current device at alloc)
  void alloc(size_t b, cudaStream_t s) {
    release();
    st = s;
    dev = cur_dev();
    cudaMemPool_t pool = lib_pool(dev);
    if (b == 0) b = 16;
    const double t0 = wall_ms();
    cudaError_t e = cudaSuccess;
    if (b >= kBigBlock) {
      size_t got = 0;
      // big blocks are quantised to 8 sizes per octave, so requests that differ slightly between
      // factorizations (a rank off by one) still map to the same cached block instead of growing the pool
      size_t q = size_t(1) << (63 - __builtin_clzll((unsigned long long)b));
      const size_t step = std::max<size_t>(q / 8, 1u << 20);
      const size_t bq = (b + step - 1) / step * step;
      p = big_cache(dev).take(bq, s, &got);
      if (!p) {
        got = bq;
        e = cudaMallocFromPoolAsync(&p, got, pool, s);
        if (e != cudaSuccess) {  // give the cached blocks back and retry once
          cudaGetLastError();
          big_cache(dev).flush(s);
          e = cudaMallocFromPoolAsync(&p, got, pool, s);
        }
        if (e != cudaSuccess) e = retry_trimmed(&p, got, s);
      }
      big = e == cudaSuccess;
      cap = got;
    } else {
      e = cudaMallocFromPoolAsync(&p, b, pool, s);
      if (e != cudaSuccess) {
        big_cache(dev).flush(s);
        e = retry_trimmed(&p, b, s);
      }
    }
    const double dt = wall_ms() - t0;
    g_ac.alloc_ms += dt;
    g_ac.alloc_max = std::max(g_ac.alloc_max, dt);
    ++g_ac.nalloc;
    if (e != cudaSuccess) {
      cudaGetLastError();
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      uint64_t res = 0, used = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      throw Error(FMMLU_ENOMEM, "device allocation of " + std::to_string(b) + " bytes failed (device free " +
                                    std::to_string(fr >> 20) + " MiB of " + std::to_string(tot >> 20) +
                                    ", library pool reserved " + std::to_string(res >> 20) + " MiB / used " +
                                    std::to_string(used >> 20) + " MiB, block cache " +
                                    std::to_string(big_cache(dev).cached() >> 20) + " MiB)");
    }
    bytes = b;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Factorization workspace per device (level block stores, M, T, W, Gram scratch): kept across
// handles so that repeated factorizations reuse the same multi-GB blocks instead of growing the
// pool (a fresh 45 GB level store stalled the host for 0.5–1.4 s on cfg5).  One factorization per
// device uses it at a time (`mu` is held for the whole fmmlu_factor); fmmlu_release_cache() frees it.
struct DevWork {
  std::mutex mu;
  DBuf slot[6];
};
DevWork& dev_work(int dev) {
  static DevWork* w[kMaxDev] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= kMaxDev) throw Error(FMMLU_ECUDA, "device ordinal out of range");
  if (!w[dev]) w[dev] = new DevWork();
  return *w[dev];
}
void release_dev_work(int dev) {
  DevWork& w = dev_work(dev);
  std::lock_guard<std::mutex> lk(w.mu);
  for (auto& d : w.slot) {
    if (d.p) d.st = nullptr;  // the last user's stream may be gone: release on the legacy stream
    d.release();
  }
}

// Pinned host staging for H2D uploads: cudaMemcpyAsync from pageable memory synchronises the
// stream first, pinned memory keeps uploads asynchronous.  Reset only after a stream sync.
struct PinnedArena {
  std::vector<std::pair<char*, size_t>> chunks;
  size_t used = 0;
  char* get(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (chunks.empty() || used + bytes > chunks.back().second) {
      size_t cap = std::max<size_t>(bytes, chunks.empty() ? (64u << 20) : 2 * chunks.back().second);
      void* p = nullptr;
      const double t0 = wall_ms();
      FMMLU_CUDA(cudaMallocHost(&p, cap));
      g_ac.pin_ms += wall_ms() - t0;
      chunks.push_back({(char*)p, cap});
      used = 0;
    }
    char* r = chunks.back().first + used;
    used += bytes;
    return r;
  }
  void reset() {  // keep the largest (last) chunk
    while (chunks.size() > 1) {
      cudaFreeHost(chunks.front().first);
      chunks.erase(chunks.begin());
    }
    used = 0;
  }
  ~PinnedArena() {
    for (auto& c : chunks) cudaFreeHost(c.first);
  }
};
thread_local PinnedArena tl_pin;

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  char* hp = tl_pin.get(bytes);
  std::memcpy(hp, src, bytes);
  FMMLU_CUDA(cudaMemcpyAsync(dst, hp, bytes, cudaMemcpyHostToDevice, st));
}

// Device staging arena for task/descriptor uploads: grow-only chunks per (thread, stream), bump
// allocation, reset after the stream has been synchronised (wait_stream) — replaces one
// cudaMallocAsync/cudaFreeAsync pair per upload (≈ 10 per elimination phase).
struct DevArena {
  std::vector<DBuf> chunks;
  size_t used = 0;
  char* get(size_t bytes, cudaStream_t st) {
    bytes = (bytes + 255) & ~size_t(255);
    if (chunks.empty() || used + bytes > chunks.back().bytes) {
      const size_t cap = std::max<size_t>(bytes, chunks.empty() ? (16u << 20) : 2 * chunks.back().bytes);
      chunks.emplace_back();
      chunks.back().alloc(cap, st);
      used = 0;
    }
    char* r = chunks.back().as<char>() + used;
    used += bytes;
    return r;
  }
  void reset() {  // the stream is idle: keep the largest (last) chunk
    while (chunks.size() > 1) chunks.erase(chunks.begin());
    used = 0;
  }
};
// per thread, never destroyed (no CUDA calls from static destructors at process exit)
thread_local std::unordered_map<cudaStream_t, DevArena>& tl_devarena = *new std::unordered_map<cudaStream_t, DevArena>();
void drop_arena(cudaStream_t st) {  // before destroying a stream: free its chunks on it while it is alive
  auto it = tl_devarena.find(st);
  if (it == tl_devarena.end()) return;
  cudaStreamSynchronize(st);
  it->second.chunks.clear();
  tl_devarena.erase(it);
}

// Collects host arrays and uploads them in one H2D copy.  With reserve_pinned(bytes) the arrays are
// collected straight into pinned staging (one host copy fewer for the large per-phase uploads).
struct Stage {
  std::vector<char> host;
  char* pin = nullptr;
  size_t pin_cap = 0, pin_used = 0;
  DBuf dev;
  void reserve_pinned(size_t bytes) {
    pin_cap = bytes + 16 * 64;
    pin = tl_pin.get(pin_cap);
    pin_used = 0;
  }
  template <class T> size_t add(const std::vector<T>& v) {
    if (pin) {
      size_t off = (pin_used + 15) & ~size_t(15);
      if (off + v.size() * sizeof(T) > pin_cap) throw Error(FMMLU_ECUDA, "staging reservation too small");
      if (!v.empty()) std::memcpy(pin + off, v.data(), v.size() * sizeof(T));
      pin_used = off + v.size() * sizeof(T);
      return off;
    }
    size_t off = (host.size() + 15) & ~size_t(15);
    host.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(host.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
  void upload(cudaStream_t s) {
    const size_t n = pin ? pin_used : host.size();
    dev.release();
    dev.p = tl_devarena[s].get(n + 16, s);
    dev.bytes = n + 16;
    dev.st = s;
    dev.borrowed = true;
    if (pin) {
      if (n) FMMLU_CUDA(cudaMemcpyAsync(dev.p, pin, n, cudaMemcpyHostToDevice, s));
    } else {
      h2d(dev.p, host.data(), host.size(), s);
    }
  }
  void upload_owned(cudaStream_t s) {  // own allocation: for data that outlives the next sync
    const size_t n = pin ? pin_used : host.size();
    dev.alloc(n + 16, s);
    if (pin) {
      if (n) FMMLU_CUDA(cudaMemcpyAsync(dev.p, pin, n, cudaMemcpyHostToDevice, s));
    } else {
      h2d(dev.p, host.data(), host.size(), s);
    }
  }
  template <class T> T* ptr(size_t off) const { return reinterpret_cast<T*>(dev.as<char>() + off); }
};

struct Phase {  // one (level, colour) elimination phase
  int level, colour;
  DBuf fac;    // complex: T | Xinv | Up | Lp per box
  DBuf idx;    // int: S | R | N per box
  DBuf recs;   // BoxRec[nrec]
  DBuf items;  // SolveItem[nitems] (row/column chunks of Lp/Up)
  int nrec = 0, kmax = 0, rmax = 0, nitems = 0;
  int tmp_rows = 0;  // Σ r over the phase's boxes (solve scratch)
  size_t fac_bytes = 0;
  DBuf ap_xs, ap_recs;  // fmmlu_apply: X_RR blocks (re-inverted X_RR⁻¹) and records pointing at them
  std::vector<BoxRec> hrecs;  // host copy of recs (multi-RHS GEMM sweeps build their problems from it)
  // separate incoming/outgoing IDs: the records of the column (unknown) side —
  // T = T_c, index lists S_c | R_c | N_c — used by the downward sweep; recs are the row side
  DBuf recs_c;
  std::vector<BoxRec> hrecs_c;
  const BoxRec* down_recs() const { return recs_c.p ? recs_c.as<BoxRec>() : recs.as<BoxRec>(); }
  const std::vector<BoxRec>& down_hrecs() const { return recs_c.p ? hrecs_c : hrecs; }
  // Sub-waves of records (boundaries into recs / items; one wave unless deterministic): no two boxes
  // of a wave share a target owner, so every atomic update of a wave lands on a distinct entry and
  // the waves run in a fixed order.  SolveItem::rec is relative to its wave's first record.
  std::vector<int> wrec{0}, witem{0};
  int nwaves() const { return (int)wrec.size() - 1; }
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Per-kernel-class device timing with CUDA events recorded on the launch stream;
// resolved at the driver's existing synchronisation points.
struct Prof {
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  double ms[16] = {}, flops[16] = {}, bytes[16] = {};
  long long launches[16] = {};
  long long total_launches = 0;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      FMMLU_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
  int begin(int cls, cudaStream_t st) {
    Rec r{cls, ev(), ev()};
    FMMLU_CUDA(cudaEventRecord(r.a, st));
    pending.push_back(r);
    return (int)pending.size() - 1;
  }
  void end(int id, cudaStream_t st) { FMMLU_CUDA(cudaEventRecord(pending[id].b, st)); }
  void add(int cls, double fl, double by, long long nl) {
    flops[cls] += fl;
    bytes[cls] += by;
    launches[cls] += nl;
    total_launches += nl;
  }
  size_t mark() const { return pending.size(); }
  // resolve the first n records (completed: the stream was synchronised after they were recorded)
  // while later ones are still in flight; their events stay checked out until the next full resolve
  void resolve_first(size_t n) {
    n = std::min(n, pending.size());
    for (size_t i = 0; i < n; ++i) {
      float t = 0.f;
      FMMLU_CUDA(cudaEventElapsedTime(&t, pending[i].a, pending[i].b));
      ms[pending[i].cls] += t;
    }
    pending.erase(pending.begin(), pending.begin() + n);
  }
  void resolve() {  // call after the stream has been synchronised
    for (auto& r : pending) {
      float t = 0.f;
      FMMLU_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.cls] += t;
    }
    pending.clear();
    used = 0;
  }
  void reset() {
    pending.clear();
    used = 0;
    for (int i = 0; i < 16; ++i) ms[i] = flops[i] = bytes[i] = 0, launches[i] = 0;
    total_launches = 0;
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

}  // namespace

// Per-level owner topology (tree-only; cached per handle): owners = level-ℓ boxes (Morton order)
// then the leaves of coarser levels (reading C7); nb[a] = owners at Chebyshev separation ≤ 2
// of owner a, including a, sorted; sep[a][i] = that separation (≤ 1: near field N, 2: Q; C6).
struct LevelTopo {
  std::vector<int> owners;
  std::vector<int> local;
  std::vector<std::vector<int>> boxN, boxQ;  // per level-ℓ box (local ids 0..nbox-1): N and Q owners
  std::vector<std::vector<int>> nb;          // per owner: block partners (pair set, sorted)
};

struct fmmlu_handle {
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  Tree tree;
  int64_t n = 0;
  DBuf geo;   // 7 × n doubles, tree order
  DBuf perm;  // int64 tree pos -> caller index
  Geo g{};
  // factor
  bool factored = false;
  double k = 0, eps = 0;
  std::vector<Phase> phases;
  DBuf root;          // n0 × n0 complex: P·A_{B_tB_t} = L·U (L unit lower, U upper; rootlu.cu)
  DBuf root_rows;     // int n0: B_t (ascending tree-order indices)
  DBuf root_rows_in;  // int n0: B_t[σ(i)], σ = the composed row interchanges (gathers P·y)
  DBuf root_dinv;     // inverses of the diagonal blocks of L and U (blocked triangular solves)
  DBuf root_flags;    // solve scratch: per row block ready flags + tickets
  // grow-only workspace slots reused by every phase / level of a factorization (borrowed, never
  // freed per phase): 0/1 level block stores by level parity, 2 M, 3 Tb, 4 W, 5 Gram G|R
  DBuf ws_slot[6];
  DBuf* ws = nullptr;  // during fmmlu_factor: the device's shared workspace (DevWork); else ws_slot
  // factor-store arena: the per-phase stores are carved from uniform chunks owned by the handle, so
  // successive factorizations reuse whole chunks from the big-block cache instead of growing the
  // stream-ordered pool for every differently sized phase store
  std::vector<DBuf> fac_chunks;
  size_t fac_used = 0;  // bytes used in the last chunk
  bool apply_ready = false;
  int tree_launches = 0;  // kernels of the last fmmlu_tree (scan, keys, 9 radix-sort passes, gather)
  int64_t n0 = 0;
  fmmlu_stats_t stats{};
  size_t cur_bytes = 0, peak_bytes = 0;
  Prof prof;
  std::vector<LevelTopo> topo;    // per-level owner topology (tree-only, cached)
  // the finished tree on the device for the owner-list kernels (devtree.cu): Morton code, leaf flag
  // and exclusive leaf count per box (level-major ids), and the level prefix on the host
  DBuf tcode, tleaf, tleafrank;
  std::vector<int> level_first;
  std::atomic<int> topo_launches{0};
  // pinned landing buffer for ranks / pivots: per thread, grow-only, never freed (pinned
  // allocations and frees per handle stalled the host for hundreds of ms)
  int* d2h(size_t n) {
    thread_local int* buf = nullptr;
    thread_local size_t cap = 0;
    if (n > cap) {
      const size_t c = std::max<size_t>(n, 2 * cap + (1u << 20));
      void* p = nullptr;
      FMMLU_CUDA(cudaMallocHost(&p, c * sizeof(int)));
      if (buf) cudaFreeHost(buf);  // only while growing (the stream was synchronised by the caller)
      buf = (int*)p;
      cap = c;
    }
    return buf;
  }
  std::vector<char> topo_ready;
  int deterministic = -1;    // 1: bitwise-reproducible factor/solve (no racing fp64 atomics); -1: env default
  int id_mode = 0;           // 0 auto, 1 Householder TSQR + CPQR, 2 Gram + pivoted Cholesky
  int gj_mode = 0;           // 0 auto (shared-memory GJ when it fits), 1 blocked panel GJ always
  int id_refine = 0;         // corrected-seminormal-equations steps on the Gram-path T (0..3)
  int pchol_mode = 0;        // 0 register-resident pivoted Cholesky (b ≤ 512), 1 shared-memory cluster kernel
  double rho_factor = 2.0;   // proxy radius / box side (reading C5)
  int pchol_ll = 1;          // Gram path, b ≤ 512: left-looking pivoted Cholesky first (0 for fmmlu_boxes: k ≈ b)
  int separate_id = 0;       // 1: separate incoming/outgoing IDs (DESIGN R12)
  bool fac_separate = false; // the stored factorization was built with separate IDs
  DBuf sep_perm;             // int n (separate IDs): unknown c ← equation sep_perm[c] between the sweeps
  // Repeated small-RHS solves (the factorization is computed once and applied to
  // many right-hand sides): from the second fmmlu_solve with the same nrhs on, the ≈ 5 launches per
  // phase of the per-box sweeps are replayed as one CUDA graph captured on persistent buffers.
  struct SolveGraph {
    cudaGraphExec_t exec = nullptr;
    int uses = 0;
  };
  std::map<int, SolveGraph> solve_graphs;  // by nrhs
  DBuf sv_y, sv_scr, sv_root;              // persistent solve buffers (their pointers are baked into the graphs)
  void drop_solve_graphs() {
    for (auto& kv : solve_graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    solve_graphs.clear();
  }
};

namespace {

// The handle's stream is non-blocking: make it wait for work already queued on the legacy default
// stream (the usual producer of caller device buffers in plain CUDA code).  Callers that write inputs
// on another stream must synchronise it, or pass it with fmmlu_set_stream (include/fmmlu.h).
void order_after_legacy(cudaStream_t st) {
  cudaEvent_t e;
  FMMLU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  FMMLU_CUDA(cudaEventRecord(e, cudaStreamLegacy));
  FMMLU_CUDA(cudaStreamWaitEvent(st, e, 0));
  FMMLU_CUDA(cudaEventDestroy(e));
}

// cudaStreamSynchronize with the blocked time accounted (stats: host vs device-wait split)
void wait_stream(fmmlu_handle* h, cudaStream_t st) {
  double t0 = now_ms();
  // spin on the stream instead of a blocking synchronize: the factorization waits here once per
  // phase for the ranks, and the blocking wake-up added tens of µs of device idle each time
  static const bool spin = !(getenv("FMMLU_BLOCKING_SYNC") && atoi(getenv("FMMLU_BLOCKING_SYNC")));
  if (spin) {
    cudaError_t e;
    while ((e = cudaStreamQuery(st)) == cudaErrorNotReady) {
    }
    FMMLU_CUDA(e);
  } else {
    FMMLU_CUDA(cudaStreamSynchronize(st));
  }
  h->stats.t_sync_wait_ms += now_ms() - t0;
  tl_pin.reset();
  auto it = tl_devarena.find(st);
  if (it != tl_devarena.end()) it->second.reset();
}

// dst ← a view of workspace slot `slot` of at least `bytes` (the slot grows by ≥ 25 % when short;
// its old block is released stream-ordered, after the work that used it)
void borrow_ws(fmmlu_handle* h, int slot, DBuf& dst, size_t bytes, cudaStream_t st) {
  DBuf& w = h->ws ? h->ws[slot] : h->ws_slot[slot];
  w.st = st;  // stream-ordered release (on growth) after this user's work
  if (!w.p || w.bytes < bytes) {
    // headroom: the shared workspace is reused by later factorizations whose sizes differ slightly
    // (a rank off by one); 10 % on top of the request avoids a multi-GB regrowth (and its pool growth)
    const size_t want = h->ws ? bytes + bytes / 10 : bytes;
    const size_t grown = std::max(want, w.bytes + w.bytes / 4);
    if (w.p && w.big && h->ws) {  // outgrown shared workspace: back to the pool, not the block cache
      cudaFreeAsync(w.p, st);
      w.p = nullptr;
      w.big = false;
      w.bytes = 0;
    }
    w.alloc(grown, st);
  }
  dst.release();
  dst.p = w.p;
  dst.bytes = bytes;
  dst.st = st;
  dst.borrowed = true;
}

constexpr size_t kFacChunk = 512u << 20;
void fac_alloc(fmmlu_handle* h, DBuf& dst, size_t bytes, cudaStream_t st) {
  bytes = (bytes + 255) & ~size_t(255);
  if (h->fac_chunks.empty() || h->fac_used + bytes > h->fac_chunks.back().bytes) {
    h->fac_chunks.emplace_back();
    h->fac_chunks.back().alloc(std::max(bytes, kFacChunk), st);
    h->fac_used = 0;
  }
  dst.release();
  dst.p = h->fac_chunks.back().as<char>() + h->fac_used;
  dst.bytes = bytes;
  dst.st = st;
  dst.borrowed = true;
  h->fac_used += bytes;
}

void track(fmmlu_handle* h, long long delta) {
  h->cur_bytes += delta;
  h->peak_bytes = std::max(h->peak_bytes, h->cur_bytes);
}

int proxy_count(double k, double rho, double eps) {
  // n_γ = 2p(p+1), p = max(8, ⌈κ + 1.8 (log10(1/ε))^{2/3} κ^{1/3}⌉), κ = kρ (reading C5)
  double kap = k * rho;
  double p = std::ceil(kap + 1.8 * std::pow(std::log10(1.0 / eps), 2.0 / 3.0) * std::cbrt(kap));
  int pi = std::max(8, (int)p);
  return 2 * pi * (pi + 1);
}

constexpr int kTile = 64;

// upper = true: only output tiles with tile-row ≤ tile-column (Hermitian results).  One group per
// problem; the 64×64 tile list is expanded on the device (gemm_run).
void add_gemm(std::vector<GemmProblem>& probs, std::vector<GemmGroup>& groups, const GemmProblem& p0,
              bool upper = false) {
  GemmProblem p = p0;
  // 32-wide output tiles for skinny plain stores (the multi-RHS solve sweeps: n = nrhs ≤ 32)
  p.bn = (p.n <= 32 && p.slot == nullptr && !upper) ? 32 : 64;
  const int cnt = gemm_tile_count(p, upper);
  if (cnt <= 0) return;
  const int first = groups.empty() ? 0 : groups.back().first + groups.back().count;
  groups.push_back(GemmGroup{(int)probs.size(), first, cnt, upper ? 1 : 0});
  probs.push_back(p);
}
// One launch needs one tile width: mixed batches fall back to 64 (tile counts recomputed).
int unify_bn(std::vector<GemmProblem>& probs, std::vector<GemmGroup>& groups) {
  if (probs.empty()) return 64;
  bool all32 = true;
  for (auto& p : probs) all32 = all32 && p.bn == 32;
  if (all32) return 32;
  int first = 0;
  for (auto& g : groups) {
    probs[g.p].bn = 64;
    g.first = first;
    g.count = gemm_tile_count(probs[g.p], g.upper != 0);
    first += g.count;
  }
  return 64;
}
long long group_tiles(const GemmGroup* g, size_t n) { return n ? (long long)g[n - 1].first + g[n - 1].count : 0; }

// Expand the groups' tiles into a stream-ordered scratch list and run the batched GEMM.
void gemm_run(const GemmProblem* d_probs, const GemmGroup* d_groups, int ngroups, long long ntiles, cplx alpha,
              int scatter, cplx* bsr, cudaStream_t st, int bn = 64) {
  if (ntiles <= 0) return;
  DBuf tb;
  tb.alloc((size_t)ntiles * sizeof(GemmTile), st);
  gemm_expand(d_probs, d_groups, ngroups, tb.as<GemmTile>(), st);
  gemm_batched(d_probs, tb.as<GemmTile>(), (int)ntiles, alpha, scatter, bsr, st, bn);
}  // tb is released in stream order after the launches

// Algorithmic work of a batch: 8mnk real flops per complex GEMM; bytes = read A and B once,
// read-modify-write C once (16 B per complex element).
void gemm_work(const std::vector<GemmProblem>& probs, double& fl, double& by) {
  fl = by = 0;
  for (auto& p : probs) {
    fl += 8.0 * p.m * (double)p.n * p.k;
    by += 16.0 * ((double)p.m * p.k + (double)p.k * p.n) + 32.0 * (double)p.m * p.n;
  }
}

void run_gemms(std::vector<GemmProblem>& probs, std::vector<GemmGroup>& tiles, cplx alpha,
               int scatter, cplx* bsr, cudaStream_t st, std::vector<DBuf>& keep, Prof& P, int cls,
               double work_scale = 1.0) {
  if (tiles.empty()) return;
  const int bn = unify_bn(probs, tiles);
  Stage s;
  size_t op = s.add(probs), ot = s.add(tiles);
  s.upload(st);
  double fl, by;
  gemm_work(probs, fl, by);
  fl *= work_scale;  // e.g. 0.5 for Hermitian products computed on upper tiles only
  by *= work_scale;
  static const bool trace = getenv("FMMLU_TRACE") != nullptr;
  if (trace && cls == FMMLU_K_SCHUR)  // per-launch algorithmic work (to pair with ncu captures)
    fprintf(stderr, "[fmmlu] schur launch: %zu boxes, %.6g flops, %.6g bytes (algorithmic)\n", probs.size(), fl, by);
  int id = P.begin(cls, st);
  gemm_run(s.ptr<GemmProblem>(op), s.ptr<GemmGroup>(ot), (int)tiles.size(), group_tiles(tiles.data(), tiles.size()),
           alpha, scatter, bsr, st, bn);
  P.end(id, st);
  P.add(cls, fl, by, 1);
  keep.push_back(std::move(s.dev));
  probs.clear();
  tiles.clear();
}

// One batch of GEMMs without profiling (the caller brackets a whole stage).
void gemm_batched_staged(std::vector<GemmProblem>& probs, std::vector<GemmGroup>& tiles, cplx alpha,
                         cudaStream_t st, std::vector<DBuf>& keep) {
  if (tiles.empty()) return;
  const int bn = unify_bn(probs, tiles);
  Stage s;
  size_t op = s.add(probs), ot = s.add(tiles);
  s.upload(st);
  gemm_run(s.ptr<GemmProblem>(op), s.ptr<GemmGroup>(ot), (int)tiles.size(), group_tiles(tiles.data(), tiles.size()),
           alpha, 0, nullptr, st, bn);
  keep.push_back(std::move(s.dev));
  probs.clear();
  tiles.clear();
}

// Root block solve / forward product on y (tree order, ld ldy), rows B_t:
// solve y[B_t] ← A_t⁻¹ y[B_t] = U⁻¹L⁻¹(P y[B_t]);  fwd y[B_t] ← A_t y[B_t] = Pᵀ(L U y[B_t]).
// yout (separate IDs: the equations live in y, the unknowns / products go to another vector; same ld)
// tbuf: caller-owned n0 × nrhs scratch (the graph-captured solve; nullptr: allocated here)
void root_solve(fmmlu_handle* h, cplx* y, int ldy, int nrhs, cudaStream_t st, cplx* yout = nullptr,
                cplx* tbuf = nullptr) {
  if (h->n0 <= 0) return;
  const int n0 = (int)h->n0;
  DBuf T;
  if (!tbuf) {
    T.alloc((size_t)n0 * nrhs * sizeof(cplx), st);
    tbuf = T.as<cplx>();
  }
  launch_rows_move(h->root_rows_in.as<int>(), n0, y, ldy, tbuf, nrhs, 0, st);
  root_lu_solve(h->root.as<cplx>(), n0, h->root_dinv.as<cplx>(), tbuf, n0, nrhs, h->root_flags.as<int>(), st);
  launch_rows_move(h->root_rows.as<int>(), n0, yout ? yout : y, ldy, tbuf, nrhs, 1, st);
}
void root_fwd(fmmlu_handle* h, cplx* y, int ldy, int nrhs, cudaStream_t st, cplx* yout = nullptr) {
  if (h->n0 <= 0) return;
  const int n0 = (int)h->n0;
  DBuf T;
  T.alloc(2 * (size_t)n0 * nrhs * sizeof(cplx), st);
  cplx* Y = T.as<cplx>();
  launch_rows_move(h->root_rows.as<int>(), n0, y, ldy, Y, nrhs, 0, st);
  root_lu_mult(h->root.as<cplx>(), n0, Y, Y + (size_t)n0 * nrhs, n0, nrhs, st);
  launch_rows_move(h->root_rows_in.as<int>(), n0, yout ? yout : y, ldy, Y, nrhs, 1, st);
}
// Separate IDs: between the sweeps the vector changes sides.  After the upward
// sweep y holds z = X_RR⁻¹t at every eliminated equation R_r; the unknown at R_c[i] is that value
// (D⁻¹ maps R_r to R_c), so y2[c] = y[sep_perm[c]], and the root solve writes y2[B_t^c].  The
// downward sweep then runs on y2 with the column-side records, and y2 is copied back.
struct SepSwap {
  DBuf y2;
  cplx* begin(fmmlu_handle* h, cplx* y, int ldy, int nrhs, cudaStream_t st) {
    if (!h->fac_separate) return nullptr;
    if (ldy != (int)h->n) throw Error(FMMLU_EINVAL, "separate IDs: the sweeps need ld = n");
    y2.alloc((size_t)h->n * nrhs * sizeof(cplx), st);
    launch_rows_move(h->sep_perm.as<int>(), (int)h->n, y, ldy, y2.as<cplx>(), nrhs, 0, st);
    return y2.as<cplx>();
  }
  void end(fmmlu_handle* h, cplx* y, int nrhs, cudaStream_t st) {
    if (!y2.p) return;
    FMMLU_CUDA(cudaMemcpyAsync(y, y2.p, (size_t)h->n * nrhs * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
  }
};

// ---------------------------------------------------------------------------- blocked GJ inverse
// In-place inverse (Gauss-Jordan, partial pivoting) of every (A, n) with lda = n: panels of nb
// columns factored in shared memory, rank-nb updates of the other columns on the DMMA GEMM.
void gj_blocked(fmmlu_handle* h, const std::vector<std::pair<cplx*, int>>& mats, int* d_status,
                std::vector<DBuf>& keep, int cls) {
  cudaStream_t st = h->stream;
  if (mats.empty()) return;
  int nmax = 1;
  for (auto& m : mats) nmax = std::max(nmax, m.second);
  // Batches of ≥ 50 matrices (cfg5 levels 4-7) run faster on the blocked path — one CTA per matrix
  // per panel and DMMA updates keep every SM busy (inv class 157 → 68 ms; 92 ms with the switch at
  // 100 or 200) — while a few matrices finish sooner resident in a cluster's registers (blocked
  // always: cfg2 10.7 → 18.5 ms, cfg3 27 → 41 ms; with the switch at 50 cfg2 stays at 10.8 ms).
  static const int gj_batch = getenv("FMMLU_GJ_BATCH") ? atoi(getenv("FMMLU_GJ_BATCH")) : 50;
  const bool big_batch = h->gj_mode == 0 && (int)mats.size() >= gj_batch && nmax >= 48;
  if (h->gj_mode == 0 && !big_batch && gj_dsm_cluster_size(nmax) > 0) {
    // whole matrices resident in (cluster) shared memory: one launch for the batch
    std::vector<GjTask> tasks;
    double fl = 0, by = 0;
    long long xs = 0;
    for (auto& m : mats) xs += 2LL * m.second + 64;  // per-task exchange scratch (cluster path)
    DBuf xb;
    xb.alloc((size_t)xs * sizeof(cplx), st);
    xs = 0;
    for (auto& m : mats) {
      GjTask t{};
      t.A = m.first;
      t.lda = m.second;
      t.n = m.second;
      t.Am = xb.as<cplx>() + xs;
      xs += 2LL * m.second + 64;
      tasks.push_back(t);
      fl += 8.0 * (double)m.second * m.second * m.second;
      by += 32.0 * (double)m.second * m.second;
    }
    Stage s;
    size_t o_t = s.add(tasks);
    s.upload(st);
    int id = h->prof.begin(cls, st);
    launch_gj_dsm(s.ptr<GjTask>(o_t), (int)tasks.size(), d_status, st, nmax);
    h->prof.end(id, st);
    h->prof.add(cls, fl, by, 1);
    keep.push_back(std::move(s.dev));
    keep.push_back(std::move(xb));
    return;
  }
  int nb = gj_panel_width(nmax);
  bool cluster_panel = false;
  static const int panel_env = getenv("FMMLU_GJ_PANEL") ? atoi(getenv("FMMLU_GJ_PANEL")) : 0;
  bool reg_panel = false;
  if (panel_env == 0 && nb < 32 && nmax > 512 && gj_panel_reg_width(nmax) >= 16) {
    // tall blocks (root): register-resident panel rows over a 16-CTA cluster, L2 exchange
    nb = gj_panel_reg_width(nmax);
    reg_panel = true;
  } else if (panel_env <= 2 && panel_env != 1 && nb < 32 && nmax > 64) {  // shared-memory cluster panel
    for (int w = 32; w >= 8; w /= 2)
      if (gj_panel_cluster_size(nmax, w) > 0) {
        nb = w;
        cluster_panel = true;
        break;
      }
  }
  long long csz = 0, isz = 0;
  for (auto& m : mats) {
    csz += 2LL * m.second * nb + (long long)m.second * m.second;
    isz += m.second;
  }
  DBuf cb, ib;
  cb.alloc((size_t)csz * sizeof(cplx), st);
  ib.alloc((size_t)std::max<long long>(isz, 1) * sizeof(int), st);
  std::vector<GjTask> tasks;
  std::vector<long long> soff;
  long long co = 0, io = 0;
  double fl = 0, by = 0;
  for (auto& m : mats) {
    GjTask t{};
    t.A = m.first;
    t.lda = m.second;
    t.n = m.second;
    t.Am = cb.as<cplx>() + co;
    co += (long long)m.second * nb;
    t.Y = cb.as<cplx>() + co;
    co += (long long)m.second * nb;
    soff.push_back(co);
    co += (long long)m.second * m.second;
    t.piv = ib.as<int>() + io;
    io += m.second;
    tasks.push_back(t);
    fl += 8.0 * (double)m.second * m.second * m.second;
    by += 32.0 * (double)m.second * m.second;
  }
  std::vector<GemmProblem> gp;
  std::vector<GemmGroup> gt;
  std::vector<std::pair<size_t, size_t>> launches;  // (group offset, group count) per panel
  std::vector<int> lbn;                             // output tile width per panel launch
  for (int j0 = 0; j0 < nmax; j0 += nb) {
    std::vector<GemmProblem> pp;
    std::vector<GemmGroup> tt;
    for (auto& t : tasks) {
      if (j0 >= t.n) continue;
      const int jb = std::min(nb, t.n - j0);
      GemmProblem L{};
      L.m = t.n;
      L.n = j0;
      L.k = jb;
      L.opA = kOpN;
      L.opB = kOpN;
      L.A = t.Am;
      L.lda = t.n;
      L.B = t.Y;
      L.ldb = nb;
      L.C = t.A;
      L.ldc = t.lda;
      add_gemm(pp, tt, L);
      GemmProblem R = L;
      R.n = t.n - j0 - jb;
      R.B = t.Y + (size_t)(j0 + jb) * nb;
      R.C = t.A + (size_t)(j0 + jb) * t.lda;
      add_gemm(pp, tt, R);
    }
    lbn.push_back(unify_bn(pp, tt));
    for (auto& x : tt) x.p += (int)gp.size();
    launches.push_back({gt.size(), tt.size()});
    gp.insert(gp.end(), pp.begin(), pp.end());
    gt.insert(gt.end(), tt.begin(), tt.end());
  }
  Stage s;
  size_t o_t = s.add(tasks), o_s = s.add(soff), o_p = s.add(gp), o_g = s.add(gt);
  s.upload(st);
  DBuf xsb;
  if (reg_panel) xsb.alloc((size_t)tasks.size() * gj_panel_reg_scratch(nb) * sizeof(cplx), st);
  int id = h->prof.begin(cls, st);
  int pi = 0;
  long long nl = 0;
  for (int j0 = 0; j0 < nmax; j0 += nb, ++pi) {
    if (reg_panel)
      launch_gj_panel_reg(s.ptr<GjTask>(o_t), (int)tasks.size(), j0, nb, d_status, xsb.as<cplx>(), st, nmax);
    else if (cluster_panel)
      launch_gj_panel_cluster(s.ptr<GjTask>(o_t), (int)tasks.size(), j0, nb, d_status, st, nmax);
    else
      launch_gj_panel(s.ptr<GjTask>(o_t), (int)tasks.size(), j0, nb, d_status, st, nmax);
    launch_gj_swap(s.ptr<GjTask>(o_t), (int)tasks.size(), j0, nb, st, nmax);
    nl += 2;
    if (launches[pi].second) {
      gemm_run(s.ptr<GemmProblem>(o_p), s.ptr<GemmGroup>(o_g) + launches[pi].first, (int)launches[pi].second,
               group_tiles(gt.data() + launches[pi].first, launches[pi].second), cmk(1.0, 0.0), 0, nullptr, st,
               lbn[pi]);
      ++nl;
    }
  }
  launch_gj_unscramble(s.ptr<GjTask>(o_t), (int)tasks.size(), cb.as<cplx>(), s.ptr<long long>(o_s), st, nmax);
  h->prof.end(id, st);
  h->prof.add(cls, fl, by, nl + 2);
  keep.push_back(std::move(s.dev));
  keep.push_back(std::move(cb));
  keep.push_back(std::move(ib));
  keep.push_back(std::move(xsb));
}

// ---------------------------------------------------------------------------- large-box pivoted Cholesky
void pchol_big(fmmlu_handle* h, cplx* G, const std::vector<long long>& goff, long long gsz,
               const std::vector<int>& bcol, const std::vector<int>& permoff, int* d_perm, int* d_k, double eps,
               std::vector<DBuf>& keep) {
  cudaStream_t st = h->stream;
  const int nbx = (int)bcol.size();
  const int NB = 32;
  int bmax = 1;
  long long cs = 0, ds = 0, is = 0;
  for (int b : bcol) {
    bmax = std::max(bmax, b);
    cs += (long long)b * b + (long long)NB * b;
    ds += b;
    is += 2LL * b;
  }
  DBuf cb, db, ib, sb;
  // at least a big block: it then comes from the quantised block cache and is reused by the next
  // factorization (as a ≈ 26 MB pool allocation of a slightly different size every time it made the
  // pool grow: one 46 ms cudaMallocAsync per cfg5 factorization, FMMLU_TRACE allocator line)
  cb.alloc(std::max<size_t>((size_t)cs * sizeof(cplx), kBigBlock), st);
  db.alloc((size_t)ds * sizeof(double), st);
  ib.alloc((size_t)is * sizeof(int), st);
  sb.alloc((size_t)nbx * sizeof(PcholState), st);
  std::vector<PcholState> states(nbx, PcholState{0, 1, 0.0});
  h2d(sb.p, states.data(), states.size() * sizeof(PcholState), st);
  std::vector<PcholBig> tasks(nbx);
  long long co = 0, dof = 0, io = 0;
  for (int j = 0; j < nbx; ++j) {
    PcholBig& t = tasks[j];
    t.G = G + goff[j];
    t.R = cb.as<cplx>() + co;
    co += (long long)bcol[j] * bcol[j];
    t.Rp = cb.as<cplx>() + co;
    co += (long long)NB * bcol[j];
    t.d = db.as<double>() + dof;
    dof += bcol[j];
    t.done = ib.as<int>() + io;
    io += bcol[j];
    t.piv = ib.as<int>() + io;
    io += bcol[j];
    t.state = sb.as<PcholState>() + j;
    t.b = bcol[j];
    t.out_off = permoff[j];
    t.kslot = j;
  }
  std::vector<GemmProblem> gp;
  std::vector<GemmGroup> gt;
  for (int j = 0; j < nbx; ++j) {
    GemmProblem P{};
    P.m = bcol[j];
    P.n = bcol[j];
    P.k = NB;
    P.opA = kOpC;
    P.opB = kOpN;
    P.A = tasks[j].Rp;
    P.lda = NB;
    P.B = tasks[j].Rp;
    P.ldb = NB;
    P.C = tasks[j].G;
    P.ldc = bcol[j];
    P.active = &tasks[j].state->active;
    add_gemm(gp, gt, P);
  }
  const int pbn = unify_bn(gp, gt);
  Stage s;
  size_t o_t = s.add(tasks), o_p = s.add(gp), o_g = s.add(gt);
  s.upload(st);
  int id = h->prof.begin(FMMLU_K_CPQR, st);
  for (int j0 = 0; j0 < bmax; j0 += NB) {
    launch_pchol_big_panel(s.ptr<PcholBig>(o_t), nbx, NB, eps, st, bmax);
    gemm_run(s.ptr<GemmProblem>(o_p), s.ptr<GemmGroup>(o_g), (int)gt.size(), group_tiles(gt.data(), gt.size()),
             cmk(-1.0, 0.0), 0, nullptr, st, pbn);
  }
  launch_pchol_big_finish(s.ptr<PcholBig>(o_t), nbx, d_perm, d_k, st, bmax);
  h->prof.end(id, st);
  h->prof.add(FMMLU_K_CPQR, 0, 0, 2 * ((bmax + NB - 1) / NB) + 1);
  keep.push_back(std::move(s.dev));
  keep.push_back(std::move(cb));
  keep.push_back(std::move(db));
  keep.push_back(std::move(ib));
  keep.push_back(std::move(sb));
  (void)gsz;
}

// ---------------------------------------------------------------------------- cluster TSQR
// Only R of M = Q R is needed (CPQR(R) selects the same pivots and T as CPQR(M): Qᴴ preserves
// column norms and inner products).  Each round splits every box matrix that does not fit one
// 16-CTA cluster into row chunks that do, factors them with the cluster Householder kernel
// (chunk resident in distributed shared memory), and stacks the triangular factors; repeat
// until the box matrix fits a cluster for the pivoted pass.  mp/mrows are updated (ld = rows).
void tsqr_cluster(fmmlu_handle* h, std::vector<cplx*>& mp, std::vector<int>& mrows, const std::vector<int>& bcol,
                  std::vector<DBuf>& keep) {
  cudaStream_t st = h->stream;
  Prof& P = h->prof;
  const int nbx = (int)mp.size();
  for (;;) {
    std::vector<int> todo;
    int bmax = 0;
    for (int j = 0; j < nbx; ++j)
      if (hqr_cluster_size(mrows[j], bcol[j]) == 0) {
        todo.push_back(j);
        bmax = std::max(bmax, bcol[j]);
      }
    if (todo.empty()) return;
    const int H = hqr_max_rows(bmax, 16);
    if (H <= bmax) throw Error(FMMLU_ENOTIMPL, "box with too many actives for the cluster TSQR");
    std::vector<long long> noff(nbx, 0);
    std::vector<int> nrows(nbx, 0);
    long long tot = 0;
    for (int j : todo) {
      const int nch = (mrows[j] + H - 1) / H, bh = mrows[j] / nch, ex = mrows[j] % nch;
      int rr = 0;
      for (int c = 0; c < nch; ++c) rr += std::min(bh + (c < ex ? 1 : 0), bcol[j]);
      if (rr >= mrows[j])
        throw Error(FMMLU_ENOTIMPL, "cluster TSQR cannot reduce a " + std::to_string(mrows[j]) + "x" +
                                        std::to_string(bcol[j]) + " ID matrix (box too large for id_mode 1)");
      noff[j] = tot;
      nrows[j] = rr;
      tot += (long long)rr * bcol[j];
    }
    DBuf next;
    next.alloc((size_t)tot * sizeof(cplx), st);
    std::vector<ClusterQrTask> tasks;
    int hmax = 1;
    double fl = 0, by = 0;
    for (int j : todo) {
      const int nch = (mrows[j] + H - 1) / H, bh = mrows[j] / nch, ex = mrows[j] % nch, b = bcol[j];
      int r0 = 0, ro = 0;
      for (int c = 0; c < nch; ++c) {
        const int hc = bh + (c < ex ? 1 : 0);
        tasks.push_back(ClusterQrTask{mp[j] + r0, next.as<cplx>() + noff[j] + ro, mrows[j], hc, b, nrows[j], 0, 0});
        r0 += hc;
        ro += std::min(hc, b);
        hmax = std::max(hmax, hc);
        const double kq = std::min(hc, b);
        fl += 8.0 * ((double)hc * b * kq - 0.5 * (hc + b) * kq * kq + kq * kq * kq / 3.0);
        by += 16.0 * hc * b + 16.0 * kq * b;
      }
    }
    Stage s;
    size_t o_t = s.add(tasks);
    s.upload(st);
    std::vector<int> tm, tb;
    for (auto& t : tasks) {
      tm.push_back(t.m);
      tb.push_back(t.b);
    }
    int id = P.begin(FMMLU_K_QR, st);
    launch_hqr_cluster(s.ptr<ClusterQrTask>(o_t), (int)tasks.size(), 0, nullptr, nullptr, 0.0, st, tm.data(),
                       tb.data());
    P.end(id, st);
    P.add(FMMLU_K_QR, fl, by, 1);
    for (int j : todo) {
      mp[j] = next.as<cplx>() + noff[j];
      mrows[j] = nrows[j];
    }
    keep.push_back(std::move(s.dev));
    keep.push_back(std::move(next));
  }
}

// ---------------------------------------------------------------------------- factorization
// N/Q lists of the level-ℓ boxes from 5×5×5 cell lookups (coarser owners found through their
// ancestors), and the block-pair set = all pairs (x, y) with x, y ∈ {B} ∪ N(B) plus (B, q), (q, B),
// q ∈ Q(B), over the level-ℓ boxes B: exactly the blocks the level can read or modify (and every
// block modified at level ℓ+1 maps into it, since both owners touch the parent box).
// Persistent host worker pool for the per-box bookkeeping loops (spawning threads per phase cost
// more than the loops themselves).  parallel_for(count, fn(lo, hi)) splits [0, count) into chunks
// run by the workers and the caller; small counts run inline.
class HostPool {
 public:
  // Two pools: 0 for the thread that runs the factorization, 1 for its ID-preparation worker, so
  // that the two do not serialise each other's loops (one parallel region at a time per pool).
  static HostPool& get(int which = 0) {
    static HostPool* p[2] = {new HostPool(), new HostPool()};  // never destroyed (workers live until process exit)
    return *p[which ? 1 : 0];
  }
  template <class F>
  void parallel_for(int count, int min_par, F&& fn) {
    const int nw = (int)workers_.size();
    // one parallel region at a time: a concurrent caller (another handle on another host thread)
    // runs its loop inline instead of sharing the workers
    std::unique_lock<std::mutex> busy(call_mu_, std::try_to_lock);
    if (nw == 0 || count < min_par || !busy.owns_lock()) {
      fn(0, count);
      return;
    }
    std::unique_lock<std::mutex> lk(m_);
    const int parts = nw + 1, chunk = (count + parts - 1) / parts;
    job_ = [&fn, chunk, count](int w) {
      const int lo = w * chunk, hi = std::min(count, lo + chunk);
      if (lo < hi) fn(lo, hi);
    };
    pending_ = nw;
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    job_(nw);  // the caller takes the last chunk
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const int n = std::max(0, std::min<int>(15, (int)std::thread::hardware_concurrency() / 2 - 1));
    for (int w = 0; w < n; ++w) workers_.emplace_back([this, w] { loop(w); });
    for (auto& t : workers_) t.detach();
  }
  void loop(int w) {
    unsigned long long seen = 0;
    for (;;) {
      std::function<void(int)> job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        job = job_;
      }
      job(w);
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  std::function<void(int)> job_;
  int pending_ = 0;
  unsigned long long gen_ = 0;
};

// Host construction of the same lists from the host tree: the FMMLU_TOPO_CHECK=1 self-check of the
// device path only (never a fallback).
void build_topo_host(const Tree& T, int lvl, LevelTopo& tp) {
  tp.owners.clear();
  for (int b : T.levels[lvl]) tp.owners.push_back(b);
  const int nlb = (int)tp.owners.size();
  for (int m = 0; m < lvl; ++m)
    for (int b : T.levels[m])
      if (T.boxes[b].leaf()) tp.owners.push_back(b);
  const int no = (int)tp.owners.size();
  tp.local.assign(T.boxes.size(), -1);
  for (int i = 0; i < no; ++i) tp.local[tp.owners[i]] = i;
  const int lim = (1 << lvl) - 1;
  // dense cell → owner grid for moderate levels (hash lookups through the ancestors otherwise)
  const bool dense = lvl <= 7;
  std::vector<int> grid;
  const int64_t side = (int64_t)1 << lvl;
  if (dense) {
    grid.assign((size_t)(side * side * side), -1);
    for (int a = 0; a < no; ++a) {
      int64_t lo[3], hi[3];
      T.extent(tp.owners[a], lvl, lo, hi);
      for (int64_t x = lo[0]; x <= hi[0]; ++x)
        for (int64_t y = lo[1]; y <= hi[1]; ++y)
          for (int64_t z = lo[2]; z <= hi[2]; ++z) grid[(size_t)((x * side + y) * side + z)] = a;
    }
  }
  tp.boxN.assign(nlb, {});
  tp.boxQ.assign(nlb, {});
  // pair set: nb[a] = ∪ { grp(i) : a ∈ grp(i) } ∪ Q-relations, grp(i) = {i} ∪ N(i).  Built as
  // per-owner lists of the groups containing it, then one stamped union per owner.  The
  // per-box classification and the per-owner unions run on a few host threads.
  const int nth = std::max(1, std::min<int>(8, (int)std::thread::hardware_concurrency() / 2));
  auto par = [&](int count, auto&& fn) {
    if (nth == 1 || count < 256) {
      fn(0, count);
      return;
    }
    std::vector<std::thread> th;
    const int chunk = (count + nth - 1) / nth;
    for (int w = 0; w < nth; ++w) {
      const int lo = w * chunk, hi = std::min(count, lo + chunk);
      if (lo < hi) th.emplace_back([&fn, lo, hi] { fn(lo, hi); });
    }
    for (auto& t : th) t.join();
  };
  par(nlb, [&](int lo, int hi) {
    std::vector<int> cand;
    for (int i = lo; i < hi; ++i) {
      const int box = tp.owners[i];
      const Box& B = T.boxes[box];
      cand.clear();
      for (int dx = -2; dx <= 2; ++dx)
        for (int dy = -2; dy <= 2; ++dy)
          for (int dz = -2; dz <= 2; ++dz) {
            const int x = B.c[0] + dx, y = B.c[1] + dy, z = B.c[2] + dz;
            if (x < 0 || y < 0 || z < 0 || x > lim || y > lim || z > lim) continue;
            int o;
            if (dense) {
              o = grid[(size_t)(((int64_t)x * side + y) * side + z)];
            } else {
              const int ob = T.owner_of_cell(lvl, x, y, z);
              o = ob >= 0 ? tp.local[ob] : -1;
            }
            if (o >= 0 && o != i) cand.push_back(o);
          }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      for (int o : cand) (T.sep(box, tp.owners[o], lvl) <= 1 ? tp.boxN[i] : tp.boxQ[i]).push_back(o);
    }
  });
  std::vector<std::vector<int>> ingrp(no), qrel(no);
  for (int i = 0; i < nlb; ++i) {
    ingrp[i].push_back(i);
    for (int x : tp.boxN[i]) ingrp[x].push_back(i);
    for (int q : tp.boxQ[i]) {
      qrel[i].push_back(q);
      qrel[q].push_back(i);
    }
  }
  tp.nb.assign(no, {});
  par(no, [&](int lo, int hi) {
    std::vector<int> stamp(no, -1);
    for (int a = lo; a < hi; ++a) {
      std::vector<int>& v = tp.nb[a];
      auto add = [&](int b2) {
        if (stamp[b2] != a) {
          stamp[b2] = a;
          v.push_back(b2);
        }
      };
      for (int i : ingrp[a]) {
        add(i);
        for (int x : tp.boxN[i]) add(x);
      }
      for (int q : qrel[a]) add(q);
      std::sort(v.begin(), v.end());
    }
  });
}

// Owner lists of one level, built on the device (devtree.cu: device_topology) from the device copy of
// the tree — owners, N (sep ≤ 1) and Q (sep 2) lists of every level box, and the block-pair set — and
// unpacked into the host containers the descriptor builders read.  Runs on its own stream (worker
// threads build the levels concurrently while the first levels are factored).
void build_topo(fmmlu_handle* h, int lvl, LevelTopo& tp) {
  const Tree& T = h->tree;
  FMMLU_CUDA(cudaSetDevice(h->dev));
  cudaStream_t st = nullptr;
  FMMLU_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DevTopo D;
  int nl = 0;
  try {
    device_topology(h->tcode.as<unsigned long long>(), h->tleaf.as<unsigned char>(), h->tleafrank.as<int>(),
                    h->level_first.data(), T.nlevels, lvl, st, D, &nl);
  } catch (...) {
    cudaStreamDestroy(st);
    throw;
  }
  FMMLU_CUDA(cudaStreamSynchronize(st));
  FMMLU_CUDA(cudaStreamDestroy(st));
  h->topo_launches += nl;
  tp.owners = std::move(D.owners);
  const int no = D.no, nlb = D.nlb;
  tp.local.assign(T.boxes.size(), -1);
  for (int i = 0; i < no; ++i) tp.local[tp.owners[i]] = i;
  tp.boxN.assign(nlb, {});
  tp.boxQ.assign(nlb, {});
  for (int i = 0; i < nlb; ++i) {
    tp.boxN[i].assign(D.nidx.begin() + D.nptr[i], D.nidx.begin() + D.nptr[i + 1]);
    tp.boxQ[i].assign(D.qidx.begin() + D.qptr[i], D.qidx.begin() + D.qptr[i + 1]);
  }
  tp.nb.assign(no, {});
  for (int a = 0; a < no; ++a) tp.nb[a].assign(D.nbidx.begin() + D.nbptr[a], D.nbidx.begin() + D.nbptr[a + 1]);
  const bool check = getenv("FMMLU_TOPO_CHECK") != nullptr;
  if (check) {  // self-check (tests): the same lists from the host tree
    LevelTopo ref;
    build_topo_host(T, lvl, ref);
    if (ref.owners != tp.owners || ref.boxN != tp.boxN || ref.boxQ != tp.boxQ || ref.nb != tp.nb)
      throw Error(FMMLU_ECUDA, "device owner lists differ from the host tree's at level " + std::to_string(lvl));
  }
}

struct LevelBSR {
  int level = -1;
  const LevelTopo* tp = nullptr;
  LevelMeta meta{};   // device CSR of the level (kept for the next level's carry-over lookups)
  DBuf meta_buf, meta_buf2;  // meta_buf2: the compacted offsets (end of the level)
  const int* d_pair_a = nullptr;  // device: owner a of every block pair (CSR order)
  int npairs = 0;
  std::vector<std::vector<int>> act;        // actives at level start (sorted), per local owner
  std::vector<std::vector<int>> actc;       // separate IDs: the active columns (same counts); else unused
  bool sep = false;
  std::vector<std::vector<long long>> poff; // complex offset of block (a, nb[a][i])
  DBuf bsr;
  long long size = 0;
  const std::vector<int>& owners() const { return tp->owners; }
  int local(int box) const { return tp->local[box]; }
  long long off(int a, int b) const {
    const std::vector<int>& v = tp->nb[a];
    auto it = std::lower_bound(v.begin(), v.end(), b);
    return (it == v.end() || *it != b) ? -1 : poff[a][it - v.begin()];
  }
};

// ID of a batch of m×b matrices M (column-major, ld m, reading C9, R4):
// perm (b ints per box at pofs[j]: skeleton first in pivot order, then the redundant columns
// ascending), k per box, T = R11⁻¹R12 (k × (b−k), ld k) at tofs[j] in Tb.  ε ≥ 1e-7 (auto):
// Gram G = MᴴM (DMMA, upper tiles + mirror) + pivoted Cholesky (cluster, or global-memory
// blocked for big b); otherwise Householder TSQR rounds + cluster CPQR.  mfin[j] = rows of the
// matrix the pivoted pass ran on (flop accounting).  May overwrite M.
struct IdAux {  // Gram path: R' = [R11 R12] over G (ld b) per box, for the refinement step
  bool gram = false;
  DBuf G;
  std::vector<long long> goff;
};

bool is_deterministic(const fmmlu_handle* h) {
  static const bool env = getenv("FMMLU_DETERMINISTIC") && atoi(getenv("FMMLU_DETERMINISTIC"));
  return h->deterministic < 0 ? env : h->deterministic != 0;
}

bool id_uses_gram(const fmmlu_handle* h, double eps, int bmax) {
  // Gram path only where its rounding cannot move the stop decision: the squared residual norms
  // carry O(b·u)·‖M‖² absolute error against the threshold ε²‖M‖² (reading R4), so require
  // ε² ≥ 4·bmax·u (ε = 1e-6 up to b ≈ 2200; ε = 1e-7 always takes the Householder path)
  return h->id_mode >= 2 || (h->id_mode == 0 && eps * eps >= 4.0 * bmax * 1.1102230246251565e-16);
}

// G_j += M_jᴴ M_j (upper 64×64 tiles; split-K with atomic accumulation where few tiles would keep
// the GPU busy) for boxes j0 ≤ j < j1.  G must be zeroed beforehand.
void gram_gemm(fmmlu_handle* h, const std::vector<cplx*>& mp, const std::vector<int>& mrows,
               const std::vector<int>& bcol, cplx* G, const std::vector<long long>& goff, int j0, int j1,
               std::vector<DBuf>& keep) {
  cudaStream_t st = h->stream;
  std::vector<GemmProblem> gp;
  std::vector<GemmGroup> gt;
  long long utiles = 0;
  for (int j = j0; j < j1; ++j) {
    const long long t = (bcol[j] + kTile - 1) / kTile;
    utiles += t * (t + 1) / 2;
  }
  static const int g_cps = getenv("FMMLU_GRAM_CPS") ? atoi(getenv("FMMLU_GRAM_CPS")) : 8;
  static const int g_minch = getenv("FMMLU_GRAM_MINCH") ? atoi(getenv("FMMLU_GRAM_MINCH")) : 128;
  const long long want = std::max<long long>(1, ((long long)g_cps * 148 + utiles - 1) / std::max<long long>(utiles, 1));
  // A ragged last block column of ≤ 32 columns (b mod 64 in 1..32) is computed with 64×32 tiles, as a
  // second, rectangular problem G[:, 64·nf ..) = Mᴴ M[:, 64·nf ..), instead of 64×64 tiles that would
  // be more than half padding (b = 200: 10 + 4·½ = 12 tile units instead of 14)
  std::vector<GemmProblem> gp32;
  std::vector<GemmGroup> gt32;
  static const bool split32 = !(getenv("FMMLU_GRAM_SPLIT32") && atoi(getenv("FMMLU_GRAM_SPLIT32")) == 0);
  for (int j = j0; j < j1; ++j) {
    const int b = bcol[j], nf = b / kTile, rem = b % kTile;
    const bool split = split32 && nf >= 1 && rem >= 1 && rem <= 32;
    GemmProblem P{};
    P.m = split ? nf * kTile : b;
    P.n = P.m;
    P.k = mrows[j];
    P.opA = kOpC;
    P.opB = kOpN;
    P.A = mp[j];
    P.lda = mrows[j];
    P.B = mp[j];
    P.ldb = mrows[j];
    P.C = G + goff[j];
    P.ldc = bcol[j];
    long long ch = (mrows[j] + want - 1) / want;
    ch = std::max<long long>(g_minch, (ch + 15) / 16 * 16);
    P.kchunk = (mrows[j] > ch && !is_deterministic(h)) ? (int)ch : 0;  // split-K adds with atomics
    add_gemm(gp, gt, P, true);  // G is Hermitian: upper tiles only, then mirrored
    if (split) {
      GemmProblem Q = P;
      Q.m = b;
      Q.n = rem;
      Q.B = mp[j] + (size_t)(nf * kTile) * mrows[j];
      Q.C = G + goff[j] + (size_t)(nf * kTile) * bcol[j];
      add_gemm(gp32, gt32, Q);  // n ≤ 32 → 32-wide tiles
    }
  }
  // (algorithmic share of the rectangular part: ½·(b + 64·nf)/b of its 8·m·b·rem flops, 0.83 … 1)
  if (!gt32.empty()) run_gemms(gp32, gt32, cmk(1.0, 0.0), 0, nullptr, st, keep, h->prof, FMMLU_K_QR, 0.9);
  run_gemms(gp, gt, cmk(1.0, 0.0), 0, nullptr, st, keep, h->prof, FMMLU_K_QR, 0.5);
}

// gram_done: the caller already accumulated G = MᴴM into workspace slot 5 (M in waves).
void id_stage(fmmlu_handle* h, std::vector<cplx*> mp, std::vector<int> mrows, const std::vector<int>& bcol,
              const std::vector<int>& pofs, const std::vector<long long>& tofs, double eps, int* permd, int* kd,
              cplx* Tb, std::vector<DBuf>& keep, std::vector<int>& mfin, IdAux* aux = nullptr,
              bool gram_done = false, bool sep_pairs = false) {
  cudaStream_t st = h->stream;
  const int nj = (int)mp.size();
  // sep_pairs (separate IDs, DESIGN R12): problems (2j, 2j+1) are the column and row side of box j.
  // The pivoting runs down to eps_stop < ε and reports the ε-rank beside it, so that both sides can
  // take k = max(k_c, k_r) from their own greedy order (k_sep_ranks); kd then holds each side's
  // final rank (smaller than k only where its pivoting stopped earlier: the host promotes there).
  DBuf keps;
  if (sep_pairs) keps.alloc((size_t)std::max(nj, 1) * sizeof(int), st);
  bool have_keps = false;
  int bmax = 1;
  for (int b : bcol) bmax = std::max(bmax, b);
  std::vector<IdTask> ids(nj);
  for (int j = 0; j < nj; ++j) {
    ids[j].Mp = nullptr;
    ids[j].m = mrows[j];
    ids[j].b = bcol[j];
    ids[j].out_off = pofs[j];
    ids[j].T = tofs[j];
  }
  const bool gram = id_uses_gram(h, eps, bmax);
  std::vector<ClusterQrTask> cq(nj);
  DBuf G;
  bool done_id = false;
  if (gram) {
    long long gsz = 0;
    std::vector<long long> goff(nj);
    for (int j = 0; j < nj; ++j) {
      goff[j] = gsz;
      gsz += (long long)bcol[j] * bcol[j];
    }
    borrow_ws(h, 5, G, 2 * (size_t)gsz * sizeof(cplx), st);  // G | R scratch
    if (!gram_done) {
      FMMLU_CUDA(cudaMemsetAsync(G.p, 0, (size_t)gsz * sizeof(cplx), st));
      gram_gemm(h, mp, mrows, bcol, G.as<cplx>(), goff, 0, nj, keep);
    }
    // the register pivoted Cholesky reads the lower triangle from the upper one itself
    const bool reg_pchol = h->id_mode != 3 && h->pchol_mode == 0 && pchol_reg_scratch(bmax) > 0;
    // ... and the left-looking kernel copies whole columns of G with the TMA engine: both triangles
    static const bool ll_env = !(getenv("FMMLU_PCHOL_LL") && atoi(getenv("FMMLU_PCHOL_LL")) == 0);
    static const int ll_min = getenv("FMMLU_PCHOL_LL_MIN") ? atoi(getenv("FMMLU_PCHOL_LL_MIN")) : 32;
    const bool want_ll = h->id_mode != 3 && ((sep_pairs && bmax <= 1024) ||
                                             (reg_pchol && ll_env && h->pchol_ll && nj >= ll_min && bmax <= 512));
    if (!reg_pchol || want_ll) {
      std::vector<cplx*> gptr(nj);
      for (int j = 0; j < nj; ++j) gptr[j] = G.as<cplx>() + goff[j];
      Stage sm;
      size_t o_gp = sm.add(gptr), o_gd = sm.add(bcol);
      sm.upload(st);
      launch_herm_mirror(sm.ptr<cplx* const>(o_gp), sm.ptr<int>(o_gd), nj, bmax, st);
      keep.push_back(std::move(sm.dev));
    }
    for (int j = 0; j < nj; ++j) {
      cq[j] = ClusterQrTask{G.as<cplx>() + goff[j], G.as<cplx>() + gsz + goff[j], bcol[j], bcol[j], bcol[j],
                            bcol[j], pofs[j], 0};
      ids[j].Mp = G.as<cplx>() + goff[j];
      ids[j].m = bcol[j];
      mfin[j] = bcol[j];
    }
    Stage s2;
    size_t o_i = s2.add(ids), o_q = s2.add(cq);
    s2.upload(st);
    int cid = h->prof.begin(FMMLU_K_CPQR, st);
    if (sep_pairs && want_ll) {
      // deeper stop, bounded by the Gram path's noise floor (R4: squared norms carry ≈ b·u·‖M‖²)
      const double eps_stop = std::min(eps, std::max(eps / 30.0, std::sqrt(4.0 * bmax * 1.1102230246251565e-16)));
      done_id = launch_pchol_ll(s2.ptr<ClusterQrTask>(o_q), nj, permd, kd, eps_stop, st, bmax, eps, keps.as<int>(),
                                true);
      have_keps = done_id;
    }
    if (!done_id && h->id_mode != 3) {
      if (reg_pchol) {  // register-resident pivoted Cholesky
        // tree path: the left-looking one-CTA-per-box kernel first (ranks stay far below b there);
        // the boxes it gives up on (k_out = −1) are taken by the register kernel behind it
        // (its gain is one box per SM instead of one per cluster: measured on cfg5 / cfg2 for minimum
        // batches of 32 / 64 / 128 boxes: cpqr class 97 / 102 / 107 ms on cfg5, 8.7-8.9 ms on cfg2)
        const bool ll = want_ll && launch_pchol_ll(s2.ptr<ClusterQrTask>(o_q), nj, permd, kd, eps, st, bmax);
        DBuf xs;
        xs.alloc((size_t)nj * pchol_reg_scratch(bmax) * sizeof(cplx), st);
        done_id = launch_pchol_reg(s2.ptr<ClusterQrTask>(o_q), nj, permd, kd, eps, xs.as<cplx>(), st, bmax, ll ? 1 : 0);
        keep.push_back(std::move(xs));
      } else {
        done_id = launch_pchol_cluster(s2.ptr<ClusterQrTask>(o_q), nj, permd, kd, eps, st, bmax);
      }
    }
    if (!done_id) {  // boxes too large for a cluster: global-memory blocked pivoted Cholesky
      pchol_big(h, G.as<cplx>(), goff, gsz, bcol, pofs, permd, kd, eps, keep);
      done_id = true;
    }
    if (have_keps) launch_sep_ranks(kd, keps.as<int>(), nj / 2, st);
    launch_trsm_T(s2.ptr<IdTask>(o_i), kd, nj, nullptr, Tb, st, bmax);
    h->prof.end(cid, st);
    h->prof.add(FMMLU_K_CPQR, 0, 0, 2);
    keep.push_back(std::move(s2.dev));
  }
  if (!done_id) {
    tsqr_cluster(h, mp, mrows, bcol, keep);
    for (int j = 0; j < nj; ++j) {
      ids[j].Mp = mp[j];
      ids[j].m = mrows[j];
      cq[j] = ClusterQrTask{mp[j], nullptr, mrows[j], mrows[j], bcol[j], 0, pofs[j], 0};
      mfin[j] = mrows[j];
    }
    Stage s2;
    size_t o_i = s2.add(ids), o_q = s2.add(cq);
    s2.upload(st);
    int cid = h->prof.begin(FMMLU_K_CPQR, st);
    if (sep_pairs) {
      launch_hqr_cluster(s2.ptr<ClusterQrTask>(o_q), nj, 1, permd, kd, eps / 30.0, st, mrows.data(), bcol.data(), eps,
                         keps.as<int>());
      launch_sep_ranks(kd, keps.as<int>(), nj / 2, st);
    } else {
      launch_hqr_cluster(s2.ptr<ClusterQrTask>(o_q), nj, 1, permd, kd, eps, st, mrows.data(), bcol.data());
    }
    launch_trsm_T(s2.ptr<IdTask>(o_i), kd, nj, nullptr, Tb, st, bmax);
    h->prof.end(cid, st);
    h->prof.add(FMMLU_K_CPQR, 0, 0, 2);
    keep.push_back(std::move(s2.dev));
  }
  if (aux && gram && done_id && h->id_mode != 1) {
    aux->gram = true;
    aux->G = std::move(G);
    aux->goff.clear();
    long long o = 0;
    for (int j = 0; j < nj; ++j) {
      aux->goff.push_back(o);
      o += (long long)bcol[j] * bcol[j];
    }
  } else {
    keep.push_back(std::move(G));
  }
  keep.push_back(std::move(keps));
}

// One corrected-seminormal-equations step for the Gram-path T (R4): E = M_R − M_S T from M
// itself (columns gathered into [S | R] order), Z = M_Sᴴ E, T += R11⁻¹ R11⁻ᴴ Z.  Brings T from
// u·cond(M_S)² to ≈ u·cond(M_S) accuracy.  Called after the ranks/pivots reached the host.
void refine_T(fmmlu_handle* h, const std::vector<cplx*>& mp, const std::vector<int>& mrows,
              const std::vector<int>& bcol, const std::vector<int>& kv, const std::vector<int>& hperm,
              const std::vector<int>& pofs, cplx* Tb, const std::vector<long long>& tofs, const IdAux& aux,
              std::vector<DBuf>& keep) {
  cudaStream_t st = h->stream;
  std::vector<int> sel;
  long long mg = 0, zs = 0;
  int kmax = 1, rmax = 0;
  for (int j = 0; j < (int)mp.size(); ++j) {
    const int kk = kv[j], r = bcol[j] - kk;
    if (kk <= 0 || r <= 0) continue;
    sel.push_back(j);
    mg += (long long)mrows[j] * bcol[j];
    zs += (long long)kk * r;
    kmax = std::max(kmax, kk);
    rmax = std::max(rmax, r);
  }
  if (sel.empty()) return;
  DBuf Mg, Zb;
  Mg.alloc((size_t)mg * sizeof(cplx), st);
  Zb.alloc((size_t)zs * sizeof(cplx), st);
  FMMLU_CUDA(cudaMemsetAsync(Zb.p, 0, (size_t)zs * sizeof(cplx), st));
  std::vector<CopyTask> cps;
  std::vector<int> maps;
  std::vector<long long> omg(mp.size()), oz(mp.size());
  long long a = 0, z = 0;
  for (int j : sel) {
    omg[j] = a;
    a += (long long)mrows[j] * bcol[j];
    oz[j] = z;
    z += (long long)kv[j] * (bcol[j] - kv[j]);
    CopyTask c{};
    c.src = mp[j] - mp[sel[0]];  // offsets relative to the first matrix (one M arena)
    c.lds = mrows[j];
    c.dst = omg[j];
    c.ldd = mrows[j];
    c.rows = mrows[j];
    c.cols = bcol[j];
    c.rmap_off = -1;
    c.cmap_off = (int)maps.size();
    maps.insert(maps.end(), hperm.begin() + pofs[j], hperm.begin() + pofs[j] + bcol[j]);
    cps.push_back(c);
  }
  split_copy_tasks(cps);
  Stage s;
  size_t o_c = s.add(cps), o_m = s.add(maps);
  s.upload(st);
  int id = h->prof.begin(FMMLU_K_CPQR, st);
  launch_copy(s.ptr<CopyTask>(o_c), (int)cps.size(), s.ptr<int>(o_m), mp[sel[0]], Mg.as<cplx>(), st);
  h->prof.end(id, st);
  std::vector<GemmProblem> gp;
  std::vector<GemmGroup> gt;
  cplx* MG = Mg.as<cplx>();
  for (int j : sel) {  // E = M_R − M_S T (in place over the gathered M_R)
    const int kk = kv[j], r = bcol[j] - kk, m = mrows[j];
    GemmProblem P{};
    P.m = m;
    P.n = r;
    P.k = kk;
    P.opA = kOpN;
    P.opB = kOpN;
    P.A = MG + omg[j];
    P.lda = m;
    P.B = Tb + tofs[j];
    P.ldb = kk;
    P.C = MG + omg[j] + (long long)kk * m;
    P.ldc = m;
    add_gemm(gp, gt, P);
  }
  run_gemms(gp, gt, cmk(-1.0, 0.0), 0, nullptr, st, keep, h->prof, FMMLU_K_QR);
  for (int j : sel) {  // Z = M_Sᴴ E
    const int kk = kv[j], r = bcol[j] - kk, m = mrows[j];
    GemmProblem P{};
    P.m = kk;
    P.n = r;
    P.k = m;
    P.opA = kOpC;
    P.opB = kOpN;
    P.A = MG + omg[j];
    P.lda = m;
    P.B = MG + omg[j] + (long long)kk * m;
    P.ldb = m;
    P.C = Zb.as<cplx>() + oz[j];
    P.ldc = kk;
    P.kchunk = m > 512 ? 256 : 0;
    add_gemm(gp, gt, P);
  }
  run_gemms(gp, gt, cmk(1.0, 0.0), 0, nullptr, st, keep, h->prof, FMMLU_K_QR);
  std::vector<RefineTask> rt;
  for (int j : sel) {
    RefineTask t{};
    t.R = aux.G.as<cplx>() + aux.goff[j];
    t.ldr = bcol[j];
    t.Z = Zb.as<cplx>() + oz[j];
    t.T = Tb + tofs[j];
    t.k = kv[j];
    t.r = bcol[j] - kv[j];
    t.kmax = kmax;
    rt.push_back(t);
  }
  Stage s2;
  size_t o_r = s2.add(rt);
  s2.upload(st);
  int id2 = h->prof.begin(FMMLU_K_CPQR, st);
  launch_refine_T(s2.ptr<RefineTask>(o_r), (int)rt.size(), kmax, rmax, st);
  h->prof.end(id2, st);
  h->prof.add(FMMLU_K_CPQR, 0, 0, 2);
  keep.push_back(std::move(s.dev));
  keep.push_back(std::move(s2.dev));
  keep.push_back(std::move(Mg));
  keep.push_back(std::move(Zb));
}

template <class J>
std::vector<int> jobs_permoff(const std::vector<J>& jobs) {
  std::vector<int> v;
  for (auto& x : jobs) v.push_back(x.permoff);
  return v;
}

void factor_impl(fmmlu_handle* h, double k, double eps) {
  cudaStream_t st = h->stream;
  Tree& T = h->tree;
  const int L = T.nlevels;
  const int n = (int)h->n;
  h->phases.clear();
  h->fac_chunks.clear();
  h->fac_used = 0;
  h->root.release();
  h->root_rows.release();
  h->root_rows_in.release();
  h->root_dinv.release();
  h->root_flags.release();
  h->apply_ready = false;
  h->factored = false;
  h->drop_solve_graphs();
  for (auto& w : h->ws_slot) w.release();
  DevWork& dw = dev_work(h->dev);
  std::lock_guard<std::mutex> dw_lock(dw.mu);  // one factorization per device uses the shared workspace
  h->ws = dw.slot;
  struct WsReset {
    fmmlu_handle* h;
    ~WsReset() {  // also on an error path: no work may still use the workspace when the lock drops
      cudaStreamSynchronize(h->stream);
      h->ws = nullptr;
    }
  } ws_reset{h};
  fmmlu_stats_t& S = h->stats;
  std::memset(S.t_levels_ms, 0, sizeof(S.t_levels_ms));
  std::memset(S.ranks_sum, 0, sizeof(S.ranks_sum));
  std::memset(S.boxes, 0, sizeof(S.boxes));
  S.n_eliminated = 0;
  S.max_rank = 0;
  S.max_b = 0;
  S.factor_bytes = 0;
  DBuf status;
  status.alloc(16, st);
  FMMLU_CUDA(cudaMemsetAsync(status.p, 0, 16, st));

  // actives per box (sorted global tree-order indices)
  std::vector<std::vector<int>> act(T.boxes.size());
  for (size_t b = 0; b < T.boxes.size(); ++b)
    if (T.boxes[b].leaf())
      for (int i = T.boxes[b].start; i < T.boxes[b].end; ++i) act[b].push_back(i);

  // separate incoming/outgoing IDs (DESIGN
  // R12): every box keeps a row skeleton S_r (row ID of the incoming matrix) and a column skeleton
  // S_c (column ID of the outgoing one) of the same size k = max(k_r, k_c).  Block (a, b) of the
  // level store is then act_r(a) × act_c(b); every "position in an owner's actives" below exists
  // once per side.  Not separate: the column-side containers alias the row-side ones.
  const bool sep = h->separate_id != 0;
  h->fac_separate = sep;
  h->sep_perm.release();
  std::vector<std::vector<int>> actc_store;
  if (sep) actc_store = act;
  std::vector<std::vector<int>>& actc = sep ? actc_store : act;
  std::vector<int> sep_pi;  // unknown (column) index → equation (row) index eliminated with it
  if (sep) {
    sep_pi.resize(n);
    for (int i = 0; i < n; ++i) sep_pi[i] = i;
  }
  std::vector<int> prevOwner(n, -1), prevPos(n, -1);  // level ℓ+1 owner (local) / position
  std::vector<int> prevPosc_store(sep ? n : 0, -1);
  std::vector<int>& prevPosc = sep ? prevPosc_store : prevPos;
  LevelBSR prev;
  std::vector<DBuf> keep;  // per-phase temporaries kept alive until the phase syncs

  // host-time trace (FMMLU_TRACE=1): sections exclusive of stream waits
  static const bool trace = getenv("FMMLU_TRACE") != nullptr;
  double tr[24] = {0};
  double tmark = now_ms(), wmark = S.t_sync_wait_ms;
  auto lap = [&](int sec) {
    double t = now_ms(), w = S.t_sync_wait_ms;
    tr[sec] += (t - tmark) - (w - wmark);
    tmark = t;
    wmark = w;
  };
  // GPU timeline markers (FMMLU_TRACE): events recorded in stream order at the stage boundaries; the
  // device time between consecutive markers is attributed to the (from, to) pair, so e.g. the gap
  // id_end → el_begin is device idle time while the host prepared the elimination.
  std::vector<std::pair<int, cudaEvent_t>> gmarks;
  auto gmark = [&](int lbl) {
    if (!trace) return;
    cudaEvent_t e;
    FMMLU_CUDA(cudaEventCreate(&e));
    FMMLU_CUDA(cudaEventRecord(e, st));
    gmarks.push_back({lbl, e});
  };
  // per-level topologies depend only on the tree: build the not-yet-cached ones concurrently
  if ((int)h->topo.size() < L) h->topo.resize(L);
  if (h->topo_ready.size() < (size_t)L) h->topo_ready.resize(L, 0);
  std::vector<std::future<void>> topo_fut(std::max(L, 1));
  for (int lvl = L - 1; lvl >= 2; --lvl)
    if (!h->topo_ready[lvl])
      topo_fut[lvl] = std::async(std::launch::async, [h, lvl] { build_topo(h, lvl, h->topo[lvl]); });
  for (int lvl = L - 1; lvl >= 2; --lvl) {
    lap(7);
    double tl0 = now_ms();
    LevelBSR cur;
    cur.level = lvl;
    if (topo_fut[lvl].valid()) topo_fut[lvl].get();  // built on a worker thread (tree-only work)
    h->topo_ready[lvl] = 1;
    cur.tp = &h->topo[lvl];
    lap(14);
    {
      const std::vector<int>& lb = T.levels[lvl];
      HostPool::get().parallel_for((int)lb.size(), 64, [&](int i0, int i1) {  // actives = ∪ children's skeletons
        std::vector<int> u;
        for (int i = i0; i < i1; ++i) {
          const int b = lb[i];
          const Box& B = T.boxes[b];
          if (B.leaf()) continue;
          u.clear();
          for (int c = 0; c < B.nchild; ++c) u.insert(u.end(), act[B.child[c]].begin(), act[B.child[c]].end());
          std::sort(u.begin(), u.end());
          act[b] = u;
          if (sep) {
            u.clear();
            for (int c = 0; c < B.nchild; ++c) u.insert(u.end(), actc[B.child[c]].begin(), actc[B.child[c]].end());
            std::sort(u.begin(), u.end());
            actc[b] = u;
          }
        }
      });
    }
    const int no = (int)cur.owners().size();
    cur.act.resize(no);
    cur.sep = sep;
    if (sep) cur.actc.resize(no);
    const std::vector<std::vector<int>>& nb = cur.tp->nb;
    cur.poff.resize(no);
    std::vector<long long> rowoff(no + 1, 0);
    HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {
      for (int a = a0; a < a1; ++a) {
        cur.act[a] = act[cur.owners()[a]];
        if (sep) cur.actc[a] = actc[cur.owners()[a]];
      }
    });
    HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {  // block-row sizes (needs every cur.act)
      for (int a = a0; a < a1; ++a) {
        long long t = 0;
        for (int b : nb[a]) t += (long long)cur.act[a].size() * cur.act[b].size();
        rowoff[a + 1] = t;
      }
    });
    for (int a = 0; a < no; ++a) rowoff[a + 1] += rowoff[a];
    const long long off = rowoff[no];
    HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {
      for (int a = a0; a < a1; ++a) {
        cur.poff[a].resize(nb[a].size());
        long long o = rowoff[a];
        for (size_t i = 0; i < nb[a].size(); ++i) {
          cur.poff[a][i] = o;
          o += (long long)cur.act[a].size() * cur.act[nb[a][i]].size();
        }
      }
    });
    cur.size = off;
    lap(15);
    // slot 0: the level's block store; slot 1: the previous level's store compacted to its skeletons
    borrow_ws(h, 0, cur.bsr, (size_t)std::max<long long>(off, 1) * sizeof(cplx), st);
    track(h, cur.bsr.bytes);

    lap(0);
    // ---- build the level's BSR (kernel entries, or carried-over Schur-updated values)
    {
      // host: flatten the level into CSR arrays (no per-pair tables; lookups happen on the device)
      std::vector<int> actoff(no + 1, 0), gidx, slot, pos, nbptr(no + 1, 0), nbidx, slptr(no + 1, 0), sllist, pair_a;
      std::vector<int> gidxc, slotc, posc;  // separate IDs: the column side
      std::vector<long long> poffv;
      std::vector<int2> tasks;
      for (int a = 0; a < no; ++a) actoff[a + 1] = actoff[a] + (int)cur.act[a].size();
      // Two passes over the owners on the host worker pool (31k owners, 2M actives, 850k block pairs
      // and 1.2M tiles on cfg5's level 7).  Pass A: per active its previous-level owner's slot and
      // position (slots numbered in order of first appearance within the owner), per owner its
      // slot list and its pair / tile counts.  Serial prefix sums.  Pass B: the pair and tile arrays.
      const int nact = actoff[no];
      gidx.resize(nact);
      slot.resize(nact);
      pos.resize(nact);
      if (sep) {
        gidxc.resize(nact);
        slotc.resize(nact);
        posc.resize(nact);
      }
      std::vector<int> slcnt(no, 0), sltmp((size_t)no * 8, -1);
      std::vector<long long> tileoff(no + 1, 0);
      std::atomic<int> bad{0};
      const bool has_prev = prev.level >= 0;
      HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {
        for (int a = a0; a < a1; ++a) {
          int* sl = &sltmp[(size_t)a * 8];
          int ns = 0;
          const int o0 = actoff[a];
          auto slot_of = [&](int po, bool may_add) {
            for (int q = 0; q < ns; ++q)
              if (sl[q] == po) return q;
            if (!may_add || ns >= 8) {
              bad = 1;
              return -1;
            }
            sl[ns] = po;
            return ns++;
          };
          const std::vector<int>& ar = cur.act[a];
          for (size_t i = 0; i < ar.size(); ++i) {
            const int g = ar[i];
            const int po = has_prev ? prevOwner[g] : -1;
            gidx[o0 + i] = g;
            slot[o0 + i] = po >= 0 ? slot_of(po, true) : -1;
            pos[o0 + i] = po >= 0 ? prevPos[g] : 0;
          }
          if (sep) {  // the same previous-level owners hold a's columns (equal counts)
            const std::vector<int>& ac = cur.actc[a];
            for (size_t i = 0; i < ac.size(); ++i) {
              const int g = ac[i];
              const int po = has_prev ? prevOwner[g] : -1;
              gidxc[o0 + i] = g;
              slotc[o0 + i] = po >= 0 ? slot_of(po, false) : -1;
              posc[o0 + i] = po >= 0 ? prevPosc[g] : 0;
            }
          }
          slcnt[a] = ns;
          const int ra = (int)ar.size();
          long long nt = 0;
          for (int b : nb[a]) nt += (long long)((ra + 63) / 64) * (((int)cur.act[b].size() + 63) / 64);
          tileoff[a + 1] = nt;
        }
      });
      if (bad) throw Error(FMMLU_ECUDA, "level build: an owner made of more than 8 previous-level owners, or a column owner without rows");
      for (int a = 0; a < no; ++a) {
        slptr[a + 1] = slptr[a] + slcnt[a];
        nbptr[a + 1] = nbptr[a] + (int)nb[a].size();
        tileoff[a + 1] += tileoff[a];
      }
      if (tileoff[no] > INT_MAX) throw Error(FMMLU_ENOTIMPL, "level build: more than 2^31 block tiles at one level");
      sllist.resize(slptr[no]);
      nbidx.resize(nbptr[no]);
      poffv.resize(nbptr[no]);
      pair_a.resize(nbptr[no]);
      tasks.resize((size_t)tileoff[no]);
      HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {
        for (int a = a0; a < a1; ++a) {
          for (int q = 0; q < slcnt[a]; ++q) sllist[slptr[a] + q] = sltmp[(size_t)a * 8 + q];
          const int ra = (int)cur.act[a].size();
          long long t = tileoff[a];
          for (size_t i = 0; i < nb[a].size(); ++i) {
            const int b = nb[a][i];
            const int p = nbptr[a] + (int)i;
            nbidx[p] = b;
            poffv[p] = cur.poff[a][i];
            pair_a[p] = a;
            const int nt = ((ra + 63) / 64) * (((int)cur.act[b].size() + 63) / 64);
            for (int q = 0; q < nt; ++q) tasks[(size_t)t++] = make_int2(p, q);
          }
        }
      });
      for (std::vector<int>* v : {&gidx, &slot, &pos, &nbidx, &sllist, &pair_a, &gidxc, &slotc, &posc})
        if (v->empty()) v->push_back(0);
      const bool nbidx_empty = poffv.empty();
      if (poffv.empty()) poffv.push_back(0);
      Stage s;  // straight into pinned staging (tens of MB on the leaf levels of cfg5)
      s.reserve_pinned(16 * 16 + sizeof(int) * (actoff.size() + gidx.size() + slot.size() + pos.size() + nbptr.size() +
                                                nbidx.size() + slptr.size() + sllist.size() + pair_a.size() +
                                                gidxc.size() + slotc.size() + posc.size()) +
                       sizeof(long long) * poffv.size() + sizeof(int2) * tasks.size());
      size_t o_ao = s.add(actoff), o_g = s.add(gidx), o_s = s.add(slot), o_p = s.add(pos), o_np = s.add(nbptr),
             o_ni = s.add(nbidx), o_po = s.add(poffv), o_sp = s.add(slptr), o_sl = s.add(sllist),
             o_pa = s.add(pair_a), o_t = s.add(tasks);
      const size_t o_gc = sep ? s.add(gidxc) : o_g, o_sc = sep ? s.add(slotc) : o_s, o_pc = sep ? s.add(posc) : o_p;
      s.upload_owned(st);  // the level CSR is read again by the next level's build
      cur.meta = LevelMeta{s.ptr<int>(o_ao), s.ptr<int>(o_g), s.ptr<int>(o_s), s.ptr<int>(o_p), s.ptr<int>(o_np),
                           s.ptr<int>(o_ni), s.ptr<long long>(o_po), s.ptr<int>(o_sp), s.ptr<int>(o_sl),
                           s.ptr<int>(o_gc), s.ptr<int>(o_sc), s.ptr<int>(o_pc)};
      int bid = h->prof.begin(FMMLU_K_BUILD, st);
      launch_build_level(s.ptr<int2>(o_t), (int)tasks.size(), s.ptr<int>(o_pa), cur.meta, prev.meta,
                         prev.level >= 0 ? 1 : 0, prev.bsr.as<cplx>(), cur.bsr.as<cplx>(), h->g, k, st);
      h->prof.end(bid, st);
      h->prof.add(FMMLU_K_BUILD, 60.0 * cur.size, 16.0 * cur.size, 1);
      cur.d_pair_a = s.ptr<int>(o_pa);
      cur.npairs = (int)poffv.size() - (nbidx_empty ? 1 : 0);
      cur.meta_buf = std::move(s.dev);
    }
    if (prev.bsr.p) track(h, -(long long)prev.bsr.bytes);
    prev.bsr.release();

    // current actives (positions within the level-start actives); ident[a]: still all of them
    std::vector<char> ident(no, 1);
    std::vector<std::vector<int>> curpos(no);
    for (int a = 0; a < no; ++a) {
      curpos[a].resize(cur.act[a].size());
      for (size_t i = 0; i < cur.act[a].size(); ++i) curpos[a][i] = (int)i;
    }
    std::vector<std::vector<int>> curposc_store;
    if (sep) curposc_store = curpos;  // positions among the level-start active columns
    std::vector<std::vector<int>>& curposc = sep ? curposc_store : curpos;
    long long total_active = 0;
    for (int a = 0; a < no; ++a) total_active += (long long)cur.act[a].size();
    const double side = T.box_side(lvl);
    const double rho = h->rho_factor * side;
    const int ngamma = proxy_count(k, rho, eps);
    const double sg = std::sqrt(4.0 * M_PI * rho * rho / ngamma);

    lap(1);
    struct BoxJob {
      int a;  // local owner index of B
      int b;
      std::vector<int> N, Q;  // local owner indices
      int nN = 0, nQ = 0;
      bool proxy = false;
      int m = 0;
      long long Moff = 0, Toff = 0;
      int permoff = 0;
      int k = 0;
      int mfin = 0;  // rows of the matrix the pivoted pass ran on
      // separate IDs: M = [M_c | M_r], each m/2 × b with ld m/2 (M_c at Moff, M_r behind it); the row
      // side uses Toff / permoff, the column side Toffc / permoffc; kr0 / kc0 = the ε-ranks of the
      // two IDs (k = their maximum)
      long long Toffc = 0;
      int permoffc = 0;
      int kr0 = 0, kc0 = 0;
      std::vector<int> keepr, keepc;  // columns of each side's T that stay redundant (see the rank read-back)
    };
    struct Cnt { int maps, cps, pts, gidx; };
    // Host-only preparation of a colour phase's ID stage (its boxes, M layout, gather and proxy
    // tasks).  It depends on the previous phase only through the current actives, so it runs on a
    // worker thread while the previous phase's elimination is prepared and launched (PAPER.md
    // L878-884: the phases of a level are sequential; only the host bookkeeping is overlapped).
    struct IdPrep {
      int colour = 8;  // 8: no further phase at this level
      std::vector<BoxJob> jobs;
      long long wsM = 0, wsT = 0;
      int permtot = 0, bmax = 0;
      bool gram_waves = false;
      std::vector<int> wave_start;
      std::vector<Cnt> at;
      std::vector<CopyTask> cps;
      std::vector<int> maps;
      std::vector<ProxyTask> pts;
      std::vector<int> gidx;
      double t_jobs = 0, t_tasks = 0;
    };
    auto prep_id = [&](int c0) -> IdPrep {
      IdPrep P;
      for (int colour = c0; colour < 8; ++colour) {
        const double t0 = now_ms();
        std::vector<BoxJob> jobs;
        {
          std::vector<int> cand;  // the colour's boxes with actives, in Morton order
          for (int bx : T.levels[lvl])
            if (T.colour(bx) == colour && !curpos[cur.local(bx)].empty()) cand.push_back(bx);
          std::vector<BoxJob> all(cand.size());
          std::vector<char> keepj(cand.size(), 0);
          HostPool::get(1).parallel_for((int)cand.size(), 64, [&](int i0, int i1) {
            for (int i = i0; i < i1; ++i) {
              const int a = cur.local(cand[i]);
              BoxJob& J = all[i];
              J.a = a;
              J.b = (int)curpos[a].size();
              for (int o : cur.tp->boxN[a])
                if (!curpos[o].empty()) {
                  J.N.push_back(o);
                  J.nN += (int)curpos[o].size();
                }
              for (int o : cur.tp->boxQ[a])
                if (!curpos[o].empty()) {
                  J.Q.push_back(o);
                  J.nQ += (int)curpos[o].size();
                }
              const long long nF = total_active - J.b - J.nN;
              if (nF == 0) continue;  // F = ∅ → S = B (reading C12)
              const long long nP = nF - J.nQ;
              J.proxy = nP > 0;
              J.m = 2 * J.nQ + (J.proxy ? 2 * ngamma : 0);
              keepj[i] = 1;
            }
          });
          for (size_t i = 0; i < all.size(); ++i)
            if (keepj[i]) jobs.push_back(std::move(all[i]));
        }
        P.t_jobs += now_ms() - t0;
        if (jobs.empty()) continue;
        const double t1 = now_ms();
        P.colour = colour;
        const int nj = (int)jobs.size();
        for (auto& J : jobs) {
          J.Moff = P.wsM;
          P.wsM += (long long)J.m * J.b;
          J.Toff = P.wsT;
          P.wsT += (long long)(J.b / 2 + 1) * (J.b - J.b / 2 + 1);
          J.permoff = P.permtot;
          P.permtot += J.b;
          if (sep) {
            J.Toffc = P.wsT;
            P.wsT += (long long)(J.b / 2 + 1) * (J.b - J.b / 2 + 1);
            J.permoffc = P.permtot;
            P.permtot += J.b;
          }
          P.bmax = std::max(P.bmax, J.b);
        }
        // Gram path: M is only needed until its Gram matrix is formed, so it is gathered in waves of
        // ≤ FMMLU_M_WAVE_GB (default 4 GB) and each wave's G_j = M_jᴴM_j accumulated before the next
        // (cfg5 level 6 would otherwise hold ≈ 30 GB of M at once).
        P.gram_waves = id_uses_gram(h, eps, P.bmax);
        P.wave_start.assign(1, 0);
        if (P.gram_waves) {
          static const double wave_gb = getenv("FMMLU_M_WAVE_GB") ? atof(getenv("FMMLU_M_WAVE_GB")) : 4.0;
          const long long cap = std::max<long long>(1, (long long)(wave_gb * 1e9 / sizeof(cplx)));
          long long w = 0, wmax = 0;
          for (int j = 0; j < nj; ++j) {
            const long long sz = (long long)jobs[j].m * jobs[j].b;
            if (w > 0 && w + sz > cap) {
              P.wave_start.push_back(j);
              w = 0;
            }
            jobs[j].Moff = w;
            w += sz;
            wmax = std::max(wmax, w);
          }
          P.wsM = wmax;
        }
        P.wave_start.push_back(nj);
        // current positions of the owners already skeletonized at this level: one table shared by
        // every box that reads them (maps[omap[o] ..]), instead of a copy per referencing box
        std::vector<int> omap(cur.owners().size(), -1);
        int tabsz = 0;
        for (const BoxJob& J : jobs)
          for (int q : J.Q)
            if (!ident[q] && omap[q] < 0) {
              omap[q] = tabsz;
              tabsz += (int)curpos[q].size();
            }
        std::vector<int> omapc_store;  // separate IDs: the same table for the column positions
        if (sep) {
          omapc_store.assign(cur.owners().size(), -1);
          for (size_t q = 0; q < omap.size(); ++q)
            if (omap[q] >= 0) {
              omapc_store[q] = tabsz;
              tabsz += (int)curposc[q].size();
            }
        }
        const std::vector<int>& omapc = sep ? omapc_store : omap;
        // pass 1: per-box offsets into every array;  pass 2: fill on the host worker pool
        std::vector<Cnt>& at = P.at;
        at.resize(nj + 1);
        {
          Cnt c{tabsz, 0, 0, 0};
          for (int j = 0; j < nj; ++j) {
            at[j] = c;
            const BoxJob& J = jobs[j];
            for (int q : J.Q) c.cps += 2 * copy_tiles((int)curpos[q].size(), J.b);
            if (J.proxy) {
              c.pts += sep ? 2 : 1;
              c.gidx += (sep ? 2 : 1) * (int)cur.act[J.a].size();
            }
          }
          at[nj] = c;
          P.maps.resize(c.maps);
          P.cps.resize(c.cps);
          P.pts.resize(c.pts);
          P.gidx.resize(c.gidx);
          for (size_t q = 0; q < omap.size(); ++q)
            if (omap[q] >= 0) std::copy(curpos[q].begin(), curpos[q].end(), P.maps.begin() + omap[q]);
          if (sep)
            for (size_t q = 0; q < omapc.size(); ++q)
              if (omapc[q] >= 0) std::copy(curposc[q].begin(), curposc[q].end(), P.maps.begin() + omapc[q]);
        }
        std::vector<CopyTask>& cps = P.cps;
        std::vector<int>& maps = P.maps;
        std::vector<ProxyTask>& pts = P.pts;
        std::vector<int>& gidx = P.gidx;
        HostPool::get(1).parallel_for(nj, 8, [&](int j0, int j1) {
          for (int j = j0; j < j1; ++j) {
            BoxJob& J = jobs[j];
            int ci = at[j].cps;
            int row = 0;
            // not separate: M = [A_QB ; A_BQᵀ ; proxy out ; proxy in] (ld m).  Separate IDs:
            // M_c = [A_QB ; proxy out] and M_r = [A_BQᵀ ; proxy in], each (m/2) × b with ld m/2
            const int mh = J.m / 2;
            const int ldm = sep ? mh : J.m;
            const long long MoffR = sep ? J.Moff + (long long)mh * J.b : J.Moff;
            for (int q : J.Q) {  // A_QB rows: block (q, B), rows restricted to q's current actives
              const int mo = omap[q];
              CopyTask c{};
              c.src = cur.off(q, J.a);
              c.lds = (int)cur.act[q].size();
              c.dst = J.Moff + row;
              c.ldd = ldm;
              c.rows = (int)curpos[q].size();
              c.cols = J.b;
              c.trans = 0;
              c.rmap_off = mo;
              c.cmap_off = -1;
              ci += emit_copy_tiles(c, &cps[ci]);
              row += c.rows;
            }
            if (sep) row = 0;
            for (int q : J.Q) {  // A_BQᵀ rows: block (B, q) transposed (q's current active columns)
              const int mo = omapc[q];
              CopyTask c{};
              c.src = cur.off(J.a, q);
              c.lds = J.b;
              c.dst = MoffR + row;
              c.ldd = ldm;
              c.rows = (int)curposc[q].size();
              c.cols = J.b;
              c.trans = 1;
              c.rmap_off = mo;
              c.cmap_off = -1;
              ci += emit_copy_tiles(c, &cps[ci]);
              row += c.rows;
            }
            if (J.proxy) {
              ProxyTask p{};
              p.dst = J.Moff;
              p.ld = ldm;
              p.row0 = row;
              p.b = J.b;
              p.idx_off = at[j].gidx;
              p.ngamma = ngamma;
              double c3[3];
              T.box_centre(cur.owners()[J.a], c3);
              p.cx = c3[0];
              p.cy = c3[1];
              p.cz = c3[2];
              p.rho = rho;
              p.sg = sg;
              if (!sep) {
                std::copy(cur.act[J.a].begin(), cur.act[J.a].end(), gidx.begin() + at[j].gidx);
                pts[at[j].pts] = p;
              } else {  // outgoing rows on B's active columns (M_c), incoming rows on its active rows (M_r)
                std::copy(cur.actc[J.a].begin(), cur.actc[J.a].end(), gidx.begin() + at[j].gidx);
                std::copy(cur.act[J.a].begin(), cur.act[J.a].end(), gidx.begin() + at[j].gidx + J.b);
                p.mode = 1;
                pts[at[j].pts] = p;
                p.mode = 2;
                p.dst = MoffR;
                p.idx_off = at[j].gidx + J.b;
                pts[at[j].pts + 1] = p;
              }
            }
          }
        });
        if (maps.empty()) maps.push_back(0);
        if (gidx.empty()) gidx.push_back(0);
        P.jobs = std::move(jobs);
        P.t_tasks = now_ms() - t1;
        return P;
      }
      return P;
    };
    IdPrep nextp = prep_id(0);
    while (nextp.colour < 8) {
      IdPrep IP = std::move(nextp);
      nextp = IdPrep{};
      const int colour = IP.colour;
      std::vector<BoxJob>& jobs = IP.jobs;
      tr[2] += IP.t_jobs;
      tr[8] += IP.t_tasks;
      lap(7);
      if (trace) {
        int bmx = 0, mmx = 0, nmx = 0;
        for (auto& J : jobs) {
          bmx = std::max(bmx, J.b);
          mmx = std::max(mmx, J.m);
          nmx = std::max(nmx, J.nN);
        }
        fprintf(stderr, "[fmmlu] L%d c%d boxes %zu bmax %d mmax %d nNmax %d ngamma %d mem %.2f GB t %.1f ms\n", lvl,
                colour, jobs.size(), bmx, mmx, nmx, ngamma, h->cur_bytes / 1e9, now_ms() - tl0);
      }
      const int nj = (int)jobs.size();
      const int permtot = IP.permtot;
      const bool gram_waves = IP.gram_waves;
      const std::vector<int>& wave_start = IP.wave_start;
      const std::vector<Cnt>& at = IP.at;

      gmark(0);
      // ------------------------------------------------ ID stage
      DBuf M, Tb, permd, kd;
      borrow_ws(h, 2, M, std::max<long long>(IP.wsM, 1) * sizeof(cplx), st);
      borrow_ws(h, 3, Tb, std::max<long long>(IP.wsT, 1) * sizeof(cplx), st);
      permd.alloc((size_t)permtot * sizeof(int), st);
      const int np = sep ? 2 * nj : nj;  // ID problems: one per box, or (column side, row side) per box
      kd.alloc((size_t)np * sizeof(int), st);
      track(h, M.bytes + Tb.bytes);
      {
        std::vector<CopyTask>& cps = IP.cps;
        std::vector<ProxyTask>& pts = IP.pts;
        Stage s;
        s.reserve_pinned(sizeof(CopyTask) * cps.size() + sizeof(int) * (IP.maps.size() + IP.gidx.size()) +
                         sizeof(ProxyTask) * pts.size());
        size_t o_c = s.add(cps), o_m = s.add(IP.maps), o_p = s.add(pts), o_g = s.add(IP.gidx);
        s.upload(st);
        lap(8);
        const int nwaves = (int)wave_start.size() - 1;
        std::vector<cplx*> mp(np);
        std::vector<int> mrows(np), bcol(np), pofs(np), mfin(np);
        std::vector<long long> tofs(np);
        for (int j = 0; j < nj; ++j) {
          if (!sep) {
            mp[j] = M.as<cplx>() + jobs[j].Moff;
            mrows[j] = jobs[j].m;
            bcol[j] = jobs[j].b;
            pofs[j] = jobs[j].permoff;
            tofs[j] = jobs[j].Toff;
          } else {  // problem 2j: column ID of M_c; 2j+1: row ID (columns of M_r)
            const int mh = jobs[j].m / 2;
            mp[2 * j] = M.as<cplx>() + jobs[j].Moff;
            mp[2 * j + 1] = M.as<cplx>() + jobs[j].Moff + (long long)mh * jobs[j].b;
            mrows[2 * j] = mrows[2 * j + 1] = mh;
            bcol[2 * j] = bcol[2 * j + 1] = jobs[j].b;
            pofs[2 * j] = jobs[j].permoffc;
            pofs[2 * j + 1] = jobs[j].permoff;
            tofs[2 * j] = jobs[j].Toffc;
            tofs[2 * j + 1] = jobs[j].Toff;
          }
        }
        DBuf Gw;
        std::vector<long long> goff(np);
        if (gram_waves) {
          long long gsz = 0;
          for (int j = 0; j < np; ++j) {
            goff[j] = gsz;
            gsz += (long long)bcol[j] * bcol[j];
          }
          borrow_ws(h, 5, Gw, 2 * (size_t)gsz * sizeof(cplx), st);  // the slot id_stage uses
          FMMLU_CUDA(cudaMemsetAsync(Gw.p, 0, (size_t)gsz * sizeof(cplx), st));
        }
        for (int w = 0; w < nwaves; ++w) {
          const int j0 = wave_start[w], j1 = wave_start[w + 1];
          int pid = h->prof.begin(FMMLU_K_GATHER, st);
          launch_copy(s.ptr<CopyTask>(o_c) + at[j0].cps, at[j1].cps - at[j0].cps, s.ptr<int>(o_m),
                      cur.bsr.as<cplx>(), M.as<cplx>(), st);
          launch_proxy(s.ptr<ProxyTask>(o_p) + at[j0].pts, at[j1].pts - at[j0].pts, s.ptr<int>(o_g), M.as<cplx>(),
                       h->g, k, st, ngamma);
          h->prof.end(pid, st);
          if (gram_waves) gram_gemm(h, mp, mrows, bcol, Gw.as<cplx>(), goff, sep ? 2 * j0 : j0, sep ? 2 * j1 : j1, keep);
        }
        {
          double by = 0, fl = 0;
          for (auto& c : cps) by += 32.0 * c.rows * c.cols;
          for (auto& p : pts) {
            const double part = p.mode ? 0.5 : 1.0;  // separate IDs: one row group per task
            by += part * 32.0 * p.ngamma * p.b;
            fl += part * 2.0 * p.ngamma * p.b * 60.0;  // ~60 flops per kernel entry (estimate)
          }
          h->prof.add(FMMLU_K_GATHER, fl, by, nwaves * ((cps.empty() ? 0 : 1) + (pts.empty() ? 0 : 1)));
        }
        keep.push_back(std::move(s.dev));
        {
          lap(9);
          id_stage(h, mp, mrows, bcol, pofs, tofs, eps, permd.as<int>(), kd.as<int>(), Tb.as<cplx>(), keep, mfin,
                   nullptr, gram_waves, sep);
          for (int j = 0; j < nj; ++j) jobs[j].mfin = sep ? mfin[2 * j] + mfin[2 * j + 1] : mfin[j];
        }
        lap(13);
      }
      gmark(1);
      std::vector<int> hk(nj), hperm(permtot);
      int* pin = h->d2h(np + permtot);
      FMMLU_CUDA(cudaMemcpyAsync(pin, kd.p, np * sizeof(int), cudaMemcpyDeviceToHost, st));
      FMMLU_CUDA(cudaMemcpyAsync(pin + np, permd.p, permtot * sizeof(int), cudaMemcpyDeviceToHost, st));
      wait_stream(h, st);
      if (!sep) {
        std::memcpy(hk.data(), pin, nj * sizeof(int));
      } else {
        for (int j = 0; j < nj; ++j) {
          jobs[j].kc0 = pin[2 * j];
          jobs[j].kr0 = pin[2 * j + 1];
        }
      }
      std::memcpy(hperm.data(), pin + np, permtot * sizeof(int));
      if (sep) {
        // k = max(k_r, k_c) so that X_{R_r R_c} is square (DESIGN R12).  The ID stage already continued
        // each side's greedy pivoting to that rank where its (deeper) stop tolerance allowed, so
        // usually k_r = k_c here.  Where a side stopped short it keeps its pivots and promotes redundant
        // columns — those that are skeletons on the other side first, so that R_r and R_c stay as
        // close as possible — to skeletons: their T columns are dropped and the remaining columns get
        // zero rows for them (the same ε-ID on a larger skeleton).  perm = [own pivots | promoted |
        // rest in the ID's order], keep = the rest's positions among the ID's redundant columns.
        HostPool::get().parallel_for(nj, 16, [&](int j0, int j1) {
          std::vector<char> mine, theirs;
          std::vector<int> np_;
          for (int j = j0; j < j1; ++j) {
            BoxJob& J = jobs[j];
            const int b = J.b;
            const int kk = std::max(J.kr0, J.kc0);
            hk[j] = kk;
            if (kk >= b) {
              hk[j] = b;
              continue;
            }
            for (int side = 0; side < 2; ++side) {
              int* own = &hperm[side == 0 ? J.permoff : J.permoffc];
              const int* oth = &hperm[side == 0 ? J.permoffc : J.permoff];
              const int k0 = side == 0 ? J.kr0 : J.kc0, ko = side == 0 ? J.kc0 : J.kr0;
              std::vector<int>& keep = side == 0 ? J.keepr : J.keepc;
              keep.clear();
              const int d = kk - k0;
              if (d == 0) {
                for (int q = 0; q < b - k0; ++q) keep.push_back(q);
                continue;
              }
              // (the other side has ko = kk pivots here and is not rewritten)
              mine.assign(b, 0);
              theirs.assign(b, 0);
              for (int i = 0; i < k0; ++i) mine[own[i]] = 1;
              for (int i = 0; i < ko; ++i) theirs[oth[i]] = 1;
              np_.assign(own, own + k0);
              int taken = 0;
              for (int q = k0; q < b && taken < d; ++q)  // the other side's skeletons first
                if (theirs[own[q]]) {
                  np_.push_back(own[q]);
                  mine[own[q]] = 1;
                  ++taken;
                }
              for (int q = k0; q < b && taken < d; ++q)
                if (!mine[own[q]]) {
                  np_.push_back(own[q]);
                  mine[own[q]] = 1;
                  ++taken;
                }
              for (int q = k0; q < b; ++q)
                if (!mine[own[q]]) {
                  keep.push_back(q - k0);
                  np_.push_back(own[q]);
                }
              std::copy(np_.begin(), np_.end(), own);
            }
          }
        });
      }
      if (trace) {
        double before[16];
        std::memcpy(before, h->prof.ms, sizeof(before));
        h->prof.resolve();
        fprintf(stderr, "[fmmlu]   gpu ms since last sync (prev elim + this ID):");
        static const char* nm[10] = {"build", "gather", "qr", "cpqr", "ef", "inv", "panel", "schur", "root", "solve"};
        for (int c = 0; c < 10; ++c)
          if (h->prof.ms[c] - before[c] > 0.005) fprintf(stderr, " %s %.3f", nm[c], h->prof.ms[c] - before[c]);
        fprintf(stderr, "\n");
      }
      // the completed events are read out after the elimination is launched (off the idle gap)
      const size_t prof_done = trace ? 0 : h->prof.mark();
      // the ID temporaries and M are freed at the end of the phase, after the elimination is
      // launched: the device is idle from here until the first elimination kernel
      std::vector<DBuf> idkeep;
      idkeep.swap(keep);
      track(h, -(long long)M.bytes);
      // update current actives: B keeps its skeleton S (sorted); then the next phase's ID stage can
      // be prepared (worker thread) while this phase's elimination is prepared and launched here
      {
        std::atomic<long long> removed{0};  // (the boxes of a phase are distinct owners: no two jobs share J.a)
        HostPool::get().parallel_for(nj, 64, [&](int j0, int j1) {
          long long rem = 0;
          for (int j = j0; j < j1; ++j) {
            BoxJob& J = jobs[j];
            J.k = hk[j];
            if (J.k == J.b) continue;
            const int* pm = &hperm[J.permoff];
            curpos[J.a].assign(pm, pm + J.k);
            std::sort(curpos[J.a].begin(), curpos[J.a].end());
            rem += J.b - J.k;
            if (sep) {
              const int* pc = &hperm[J.permoffc];
              curposc[J.a].assign(pc, pc + J.k);
              std::sort(curposc[J.a].begin(), curposc[J.a].end());
            }
            ident[J.a] = 0;
          }
          removed += rem;
        });
        total_active -= removed.load();
      }
      std::future<IdPrep> next_fut = std::async(std::launch::async, prep_id, colour + 1);

      lap(3);
      // ------------------------------------------------ elimination stage
      std::vector<int> el;  // jobs with r > 0
      for (int j = 0; j < nj; ++j) {
        jobs[j].k = hk[j];
        int r = jobs[j].b - hk[j];
        {  // CPQR on m'×b + T: 8(m'bk − (m'+b)k²/2 + k³/3) + 4k²r real flops
          double b_ = jobs[j].b, k_ = hk[j], m_ = jobs[j].mfin;
          h->prof.add(FMMLU_K_CPQR,
                      8.0 * (m_ * b_ * k_ - 0.5 * (m_ + b_) * k_ * k_ + k_ * k_ * k_ / 3.0) + 4.0 * k_ * k_ * r,
                      16.0 * m_ * b_, 0);
        }
        S.ranks_sum[lvl] += hk[j];
        S.boxes[lvl] += 1;
        S.max_rank = std::max(S.max_rank, hk[j]);
        S.max_b = std::max(S.max_b, jobs[j].b);
        if (r > 0) el.push_back(j);
      }
      if (!el.empty()) {
        Phase ph;
        ph.level = lvl;
        ph.colour = colour;
        if (is_deterministic(h)) {
          // greedy sub-waves: a box joins the first wave none of whose boxes shares an owner of
          // {B} ∪ N(B) with it (its Schur update and solve scatters then never race); the boxes are
          // reordered wave by wave (stable), so records stay contiguous per wave
          std::vector<std::vector<char>> used;
          std::vector<int> wv(el.size());
          for (size_t e = 0; e < el.size(); ++e) {
            const BoxJob& J = jobs[el[e]];
            int w = 0;
            for (;; ++w) {
              if (w == (int)used.size()) used.emplace_back(no, 0);
              bool ok = !used[w][J.a];
              for (int o : J.N) ok = ok && !used[w][o];
              if (ok) break;
            }
            used[w][J.a] = 1;
            for (int o : J.N) used[w][o] = 1;
            wv[e] = w;
          }
          std::vector<int> order(el.size());
          for (size_t e = 0; e < el.size(); ++e) order[e] = (int)e;
          std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return wv[x] < wv[y]; });
          std::vector<int> el2(el.size());
          for (size_t e = 0; e < el.size(); ++e) el2[e] = el[order[e]];
          for (size_t e = 0; e < el.size(); ++e)
            if (e == 0 || wv[order[e]] != wv[order[e - 1]]) {
              if (e) ph.wrec.push_back((int)e);
            }
          el.swap(el2);
        }
        ph.wrec.push_back((int)el.size());
        // sizes
        long long wsW = 0, facsz = 0;
        int idxsz = 0;
        std::vector<long long> WBoff(nj), WNoff(nj);
        std::vector<BoxRec> recs;
        std::vector<BoxRec> recsc;  // separate IDs: the column-side records (T_c, S_c | R_c | N_c)
        for (int j : el) {
          BoxJob& J = jobs[j];
          int r = J.b - J.k, kk = J.k, kn = kk + J.nN;
          WBoff[j] = wsW;
          wsW += (long long)J.b * (J.b + J.nN);
          WNoff[j] = wsW;
          wsW += (long long)J.nN * J.b;
          BoxRec R{};
          R.k = kk;
          R.r = r;
          R.nN = J.nN;
          R.T = facsz;
          facsz += (long long)kk * r;
          BoxRec Rc{};
          if (sep) {
            Rc.T = facsz;  // T_c (k × r)
            facsz += (long long)kk * r;
          }
          R.Xi = facsz;
          facsz += (long long)r * r;
          R.Up = facsz;
          facsz += (long long)r * kn;
          R.Lp = facsz;
          facsz += (long long)kn * r;
          R.idxS = idxsz;
          idxsz += kk;
          R.idxR = idxsz;
          idxsz += r;
          R.idxN = idxsz;
          idxsz += J.nN;
          R.tmp = ph.tmp_rows;
          ph.tmp_rows += r;
          recs.push_back(R);
          if (sep) {
            const long long tc = Rc.T;
            Rc = R;
            Rc.T = tc;
            Rc.idxS = idxsz;
            idxsz += kk;
            Rc.idxR = idxsz;
            idxsz += r;
            Rc.idxN = idxsz;
            idxsz += J.nN;
            recsc.push_back(Rc);
          }
          ph.kmax = std::max(ph.kmax, kk);
          ph.rmax = std::max(ph.rmax, r);
          S.n_eliminated += 1;
        }
        lap(16);
        DBuf W;
        if (trace) {
          int hist[5] = {0, 0, 0, 0, 0}, kmx = 0, nnmx = 0;
          for (int j : el) {
            const int r = jobs[j].b - jobs[j].k;
            hist[r <= 32 ? 0 : r <= 64 ? 1 : r <= 119 ? 2 : r <= 200 ? 3 : 4]++;
            kmx = std::max(kmx, jobs[j].k);
            nnmx = std::max(nnmx, jobs[j].nN);
          }
          fprintf(stderr,
                  "[fmmlu]   elim: boxes %zu rmax %d kmax %d nNmax %d r-hist[<=32,<=64,<=119,<=200,>200] %d %d %d %d %d "
                  "W %.2f GB factor %.2f GB\n",
                  el.size(), ph.rmax, kmx, nnmx, hist[0], hist[1], hist[2], hist[3], hist[4], wsW * 16e-9,
                  facsz * 16e-9);
        }
        borrow_ws(h, 4, W, (size_t)std::max<long long>(wsW, 1) * sizeof(cplx), st);
        fac_alloc(h, ph.fac, (size_t)std::max<long long>(facsz, 1) * sizeof(cplx), st);
        FMMLU_CUDA(cudaMemsetAsync(ph.fac.p, 0, ph.fac.bytes, st));
        ph.idx.alloc((size_t)std::max(idxsz, 1) * sizeof(int), st);
        ph.fac_bytes = ph.fac.bytes + ph.idx.bytes;
        track(h, W.bytes + ph.fac.bytes + ph.idx.bytes);
        S.factor_bytes += ph.fac.bytes + ph.idx.bytes;
        cplx* Wp = W.as<cplx>();
        cplx* F = ph.fac.as<cplx>();
        lap(17);

        std::vector<CopyTask> cps, cpsT, cpsX;
        std::vector<int> maps, hidx(idxsz);
        std::vector<int> fslot, fpos, fbld;
        std::vector<long long> ftab;
        std::vector<long long> gjoff;
        std::vector<int> gjdim;
        struct FrameRef { int slot_off, tab_off, bld_off, ns; };
        std::vector<FrameRef> frames(el.size());
        // current positions of already-skeletonized neighbour owners: one shared table (as in the ID)
        std::vector<int> nmap(no, -1);
        int ntab = 0;
        for (int j : el)
          for (int o : jobs[j].N)
            if (!ident[o] && nmap[o] < 0) {
              nmap[o] = ntab;
              ntab += (int)curpos[o].size();
            }
        std::vector<int> nmapc_store;
        if (sep) {
          nmapc_store.assign(no, -1);
          for (int o = 0; o < no; ++o)
            if (nmap[o] >= 0) {
              nmapc_store[o] = ntab;
              ntab += (int)curposc[o].size();
            }
        }
        const std::vector<int>& nmapc = sep ? nmapc_store : nmap;
        // pass 1 (serial, O(|N|) per box): where each box's entries go in every array
        struct Counts { int maps, cps, cpsT, cpsX, fs, tab, bld; };
        std::vector<Counts> at(el.size() + 1);
        {
          Counts c{ntab, 0, 0, 0, 0, 0, 0};
          for (size_t e = 0; e < el.size(); ++e) {
            at[e] = c;
            const BoxJob& J = jobs[el[e]];
            const int ns = 1 + (int)J.N.size();
            const int r = J.b - J.k;
            int nm = J.b, nf = J.k, nc = copy_tiles(J.b, J.b);
            for (int o : J.N) {
              const int no_ = (int)curpos[o].size();
              nf += no_;
              nc += copy_tiles(J.b, no_) + copy_tiles(no_, J.b);
            }
            c.maps += sep ? 2 * nm + 2 * r : nm;
            c.cps += nc;  // in 64×64 tiles (split here rather than by a serial pass afterwards)
            if (!sep) {
              c.cpsT += (J.k > 0 && r > 0) ? copy_tiles(J.k, r) : 0;
            } else {
              c.cpsT += (J.kr0 > 0 && r > 0) ? copy_tiles(J.kr0, r) : 0;
              c.cpsT += (J.kc0 > 0 && r > 0) ? copy_tiles(J.kc0, r) : 0;
            }
            c.cpsX += copy_tiles(r, r) + copy_tiles(J.k, r) + copy_tiles(J.nN, r);
            c.fs += sep ? 2 * nf : nf;
            c.tab += ns * ns;
            c.bld += ns;
          }
          at[el.size()] = c;
          maps.resize(c.maps);
          cps.resize(c.cps);
          cpsT.resize(c.cpsT);
          cpsX.resize(c.cpsX);
          gjoff.resize(el.size());
          gjdim.resize(el.size());
          fslot.resize(c.fs);
          fpos.resize(c.fs);
          ftab.resize(c.tab);
          fbld.resize(c.bld);
          for (int o = 0; o < no; ++o)
            if (nmap[o] >= 0) std::copy(curpos[o].begin(), curpos[o].end(), maps.begin() + nmap[o]);
          if (sep)
            for (int o = 0; o < no; ++o)
              if (nmapc[o] >= 0) std::copy(curposc[o].begin(), curposc[o].end(), maps.begin() + nmapc[o]);
        }
        // pass 2 (host worker pool): fill
        HostPool::get().parallel_for((int)el.size(), 8, [&](int e0, int e1) {
          for (int e = e0; e < e1; ++e) {
            BoxJob& J = jobs[el[e]];
            BoxRec& R = recs[e];
            const int kk = J.k, r = R.r, b = J.b;
            const int* pm = &hperm[J.permoff];
            int mi = at[e].maps, ci = at[e].cps;
            // local order [R | S] of B's rows and columns (separate IDs: [R_r | S_r] and [R_c | S_c])
            const int rf = mi;
            for (int i = kk; i < b; ++i) maps[mi++] = pm[i];
            for (int i = 0; i < kk; ++i) maps[mi++] = pm[i];
            const int cf = sep ? mi : rf;
            if (sep) {
              const int* pc = &hperm[J.permoffc];
              for (int i = kk; i < b; ++i) maps[mi++] = pc[i];
              for (int i = 0; i < kk; ++i) maps[mi++] = pc[i];
            }
            // W_B = [A_BB | A_BN] (rows/cols of B in [R|S] order), W_N = A_NB
            CopyTask c{};
            c.src = cur.off(J.a, J.a);
            c.lds = b;
            c.dst = WBoff[el[e]];
            c.ldd = b;
            c.rows = b;
            c.cols = b;
            c.trans = 0;
            c.rmap_off = rf;
            c.cmap_off = cf;
            ci += emit_copy_tiles(c, &cps[ci]);
            int noff = 0;
            for (int o : J.N) {
              const int mo = nmap[o], moc = nmapc[o];
              const int no_ = (int)curpos[o].size();
              CopyTask a{};
              a.src = cur.off(J.a, o);
              a.lds = b;
              a.dst = WBoff[el[e]] + (long long)(b + noff) * b;
              a.ldd = b;
              a.rows = b;
              a.cols = no_;
              a.trans = 0;
              a.rmap_off = rf;
              a.cmap_off = moc;
              ci += emit_copy_tiles(a, &cps[ci]);
              CopyTask d{};
              d.src = cur.off(o, J.a);
              d.lds = (int)cur.act[o].size();
              d.dst = WNoff[el[e]] + noff;
              d.ldd = std::max(J.nN, 1);
              d.rows = no_;
              d.cols = b;
              d.trans = 0;
              d.rmap_off = mo;
              d.cmap_off = cf;
              ci += emit_copy_tiles(d, &cps[ci]);
              noff += no_;
            }
            // T → factor store (k × r)
            if (!sep) {
              if (kk > 0 && r > 0) {
                CopyTask t{};
                t.src = J.Toff;
                t.lds = kk;
                t.dst = R.T;
                t.ldd = kk;
                t.rows = kk;
                t.cols = r;
                t.trans = 0;
                t.rmap_off = -1;
                t.cmap_off = -1;
                emit_copy_tiles(t, &cpsT[at[e].cpsT]);
              }
            } else {
              // the ID of a side returned T' (k' × (b − k')): its columns that stay redundant (keep) go
              // to rows 0..k'-1 of the k × r slot; the rows of the promoted columns stay zero (cleared store)
              int ti = at[e].cpsT;
              for (int side = 0; side < 2; ++side) {
                const int k0 = side == 0 ? J.kr0 : J.kc0;
                const std::vector<int>& keepv = side == 0 ? J.keepr : J.keepc;
                std::copy(keepv.begin(), keepv.end(), maps.begin() + mi);
                const int ko = mi;
                mi += r;
                if (k0 <= 0 || r <= 0) continue;
                CopyTask t{};
                t.src = side == 0 ? J.Toff : J.Toffc;
                t.lds = k0;
                t.dst = side == 0 ? R.T : recsc[e].T;
                t.ldd = kk;
                t.rows = k0;
                t.cols = r;
                t.trans = 0;
                t.rmap_off = -1;
                t.cmap_off = ko;
                ti += emit_copy_tiles(t, &cpsT[ti]);
              }
            }
            // X_RR → Xinv slot (after E/F)
            CopyTask x{};
            x.src = WBoff[el[e]];
            x.lds = b;
            x.dst = R.Xi;
            x.ldd = r;
            x.rows = r;
            x.cols = r;
            x.trans = 0;
            x.rmap_off = -1;
            x.cmap_off = -1;
            int xi = at[e].cpsX;
            xi += emit_copy_tiles(x, &cpsX[xi]);
            // X_{(S∪N)R} → the Lp slot: the factor keeps X_{(S∪N)R} itself (the solve applies it to
            // X_RR⁻¹ t, and the Schur update is X_{(S∪N)R}·Up), so no Lp = X_{(S∪N)R} X_RR⁻¹ product
            CopyTask xs{};
            xs.src = WBoff[el[e]] + r;  // rows S of W_B (after E/F), columns R
            xs.lds = b;
            xs.dst = R.Lp;
            xs.ldd = kk + J.nN;
            xs.rows = kk;
            xs.cols = r;
            xs.rmap_off = -1;
            xs.cmap_off = -1;
            xi += emit_copy_tiles(xs, &cpsX[xi]);
            CopyTask xn{};
            xn.src = WNoff[el[e]];  // W_N = X_{N,B}: columns R
            xn.lds = std::max(J.nN, 1);
            xn.dst = R.Lp + kk;
            xn.ldd = kk + J.nN;
            xn.rows = J.nN;
            xn.cols = r;
            xn.rmap_off = -1;
            xn.cmap_off = -1;
            emit_copy_tiles(xn, &cpsX[xi]);
            gjoff[e] = R.Xi;
            gjdim[e] = r;
          }
        });
        // pass 3 (host worker pool, built while the device runs the gathers, E/F, X_RR⁻¹ and Up of
        // this phase): the Schur scatter frames and the factor's index lists
        auto fill_frames = [&]() {
        HostPool::get().parallel_for((int)el.size(), 8, [&](int e0, int e1) {
          for (int e = e0; e < e1; ++e) {
            BoxJob& J = jobs[el[e]];
            BoxRec& R = recs[e];
            const int kk = J.k, r = R.r;
            const int* pm = &hperm[J.permoff];
            int fi = at[e].fs;
            const std::vector<int>& aB = cur.act[J.a];
            for (int i = 0; i < kk; ++i) hidx[R.idxS + i] = aB[pm[i]];
            for (int i = 0; i < r; ++i) hidx[R.idxR + i] = aB[pm[kk + i]];
            {
              int noff = 0;
              for (int o : J.N) {
                const int no_ = (int)curpos[o].size();
                for (int i = 0; i < no_; ++i) hidx[R.idxN + noff + i] = cur.act[o][curpos[o][i]];
                noff += no_;
              }
            }
            if (sep) {
              const BoxRec& Rc = recsc[e];
              const int* pc = &hperm[J.permoffc];
              const std::vector<int>& cB = cur.actc[J.a];
              for (int i = 0; i < kk; ++i) hidx[Rc.idxS + i] = cB[pc[i]];
              for (int i = 0; i < r; ++i) {
                hidx[Rc.idxR + i] = cB[pc[kk + i]];
                sep_pi[cB[pc[kk + i]]] = aB[pm[kk + i]];  // unknown R_c[i] ← equation R_r[i] (D⁻¹ block)
              }
              int noff = 0;
              for (int o : J.N) {
                const int no_ = (int)curposc[o].size();
                for (int i = 0; i < no_; ++i) hidx[Rc.idxN + noff + i] = cur.actc[o][curposc[o][i]];
                noff += no_;
              }
            }
            // scatter frame: [S | N] -> (slot, pos); slot 0 = B, slot 1+i = N[i]
            FrameRef fr;
            fr.slot_off = fi;
            fr.ns = 1 + (int)J.N.size();
            for (int i = 0; i < kk; ++i) {
              fslot[fi] = 0;
              fpos[fi++] = pm[i];
            }
            for (size_t i = 0; i < J.N.size(); ++i)
              for (int p : curpos[J.N[i]]) {
                fslot[fi] = 1 + (int)i;
                fpos[fi++] = p;
              }
            if (sep) {  // the column frame follows the row frame (col0 = k + |N|)
              const int* pc = &hperm[J.permoffc];
              for (int i = 0; i < kk; ++i) {
                fslot[fi] = 0;
                fpos[fi++] = pc[i];
              }
              for (size_t i = 0; i < J.N.size(); ++i)
                for (int p : curposc[J.N[i]]) {
                  fslot[fi] = 1 + (int)i;
                  fpos[fi++] = p;
                }
            }
            fr.tab_off = at[e].tab;
            int ti = at[e].tab;
            for (int s1 = 0; s1 < fr.ns; ++s1) {
              const int o1 = s1 == 0 ? J.a : J.N[s1 - 1];
              for (int s2 = 0; s2 < fr.ns; ++s2) ftab[ti++] = cur.off(o1, s2 == 0 ? J.a : J.N[s2 - 1]);
            }
            fr.bld_off = at[e].bld;
            for (int s1 = 0; s1 < fr.ns; ++s1) fbld[at[e].bld + s1] = (int)cur.act[s1 == 0 ? J.a : J.N[s1 - 1]].size();
            frames[e] = fr;
          }
        });
        if (fslot.empty()) { fslot.push_back(0); fpos.push_back(0); }
        if (ftab.empty()) ftab.push_back(-1);
        if (fbld.empty()) fbld.push_back(0);
        };
        // on its own host thread (with the worker pool, idle from here on) while this thread uploads
        // the descriptors and launches the gathers, E/F, X_RR⁻¹ and Up; joined before the Schur launch
        std::future<void> frames_fut = std::async(std::launch::async, fill_frames);
        if (maps.empty()) maps.push_back(0);
        lap(18);
        Stage s;
        s.reserve_pinned(16 * 8 + sizeof(CopyTask) * (cps.size() + cpsT.size() + cpsX.size()) +
                         sizeof(int) * (maps.size() + gjdim.size()) + sizeof(long long) * gjoff.size() +
                         sizeof(BoxRec) * recs.size());
        size_t o_c = s.add(cps), o_ct = s.add(cpsT), o_cx = s.add(cpsX), o_m = s.add(maps), o_go = s.add(gjoff),
               o_gd = s.add(gjdim), o_rec = s.add(recs);
        s.upload(st);
        gmark(2);
        int gid = h->prof.begin(FMMLU_K_GATHER, st);
        launch_copy(s.ptr<CopyTask>(o_c), (int)cps.size(), s.ptr<int>(o_m), cur.bsr.as<cplx>(), Wp, st);
        launch_copy(s.ptr<CopyTask>(o_ct), (int)cpsT.size(), s.ptr<int>(o_m), Tb.as<cplx>(), F, st);
        h->prof.end(gid, st);
        {
          double by = 0;
          for (auto& c : cps) by += 32.0 * c.rows * c.cols;
          for (auto& c : cpsT) by += 32.0 * c.rows * c.cols;
          h->prof.add(FMMLU_K_GATHER, 0, by, 1 + (cpsT.empty() ? 0 : 1));
        }
        lap(19);
        // E: W_B[R,:] −= Tᵀ W_B[S,:]
        std::vector<GemmProblem> gp;
        std::vector<GemmGroup> gt;
        const cplx m1 = cmk(-1.0, 0.0), p1 = cmk(1.0, 0.0);
        for (size_t e = 0; e < el.size(); ++e) {
          BoxJob& J = jobs[el[e]];
          BoxRec& R = recs[e];
          GemmProblem P{};
          P.m = R.r;
          P.n = J.b + J.nN;
          P.k = R.k;
          P.opA = kOpT;
          P.opB = kOpN;
          P.A = F + R.T;
          P.lda = std::max(R.k, 1);
          P.B = Wp + WBoff[el[e]] + R.r;
          P.ldb = J.b;
          P.C = Wp + WBoff[el[e]];
          P.ldc = J.b;
          add_gemm(gp, gt, P);
        }
        run_gemms(gp, gt, m1, 0, nullptr, st, keep, h->prof, FMMLU_K_EF);
        // F: W_B[:,R] −= W_B[:,S] T ;  W_N[:,R] −= W_N[:,S] T
        for (size_t e = 0; e < el.size(); ++e) {
          BoxJob& J = jobs[el[e]];
          BoxRec& R = recs[e];
          GemmProblem P{};
          P.m = J.b;
          P.n = R.r;
          P.k = R.k;
          P.opA = kOpN;
          P.opB = kOpN;
          P.A = Wp + WBoff[el[e]] + (long long)R.r * J.b;
          P.lda = J.b;
          P.B = F + (sep ? recsc[e].T : R.T);  // T_c on the column side
          P.ldb = std::max(R.k, 1);
          P.C = Wp + WBoff[el[e]];
          P.ldc = J.b;
          add_gemm(gp, gt, P);
          if (J.nN > 0) {
            GemmProblem Q = P;
            Q.m = J.nN;
            Q.A = Wp + WNoff[el[e]] + (long long)R.r * J.nN;
            Q.lda = J.nN;
            Q.C = Wp + WNoff[el[e]];
            Q.ldc = J.nN;
            add_gemm(gp, gt, Q);
          }
        }
        run_gemms(gp, gt, m1, 0, nullptr, st, keep, h->prof, FMMLU_K_EF);
        lap(20);
        // X_RR⁻¹ (Gauss-Jordan with partial pivoting)
        launch_copy(s.ptr<CopyTask>(o_cx), (int)cpsX.size(), s.ptr<int>(o_m), Wp, F, st);
        {
          std::vector<std::pair<cplx*, int>> mats;
          for (size_t e = 0; e < gjdim.size(); ++e) mats.push_back({F + gjoff[e], gjdim[e]});
          gj_blocked(h, mats, status.as<int>(), keep, FMMLU_K_INV);
        }
        // Up = X_RR⁻¹ X_{R(S∪N)}
        for (size_t e = 0; e < el.size(); ++e) {
          BoxJob& J = jobs[el[e]];
          BoxRec& R = recs[e];
          const int kn = R.k + J.nN;
          GemmProblem P{};
          P.m = R.r;
          P.n = kn;
          P.k = R.r;
          P.opA = kOpN;
          P.opB = kOpN;
          P.A = F + R.Xi;
          P.lda = R.r;
          P.B = Wp + WBoff[el[e]] + (long long)R.r * J.b;
          P.ldb = J.b;
          P.C = F + R.Up;
          P.ldc = R.r;
          add_gemm(gp, gt, P);
        }
        run_gemms(gp, gt, p1, 0, nullptr, st, keep, h->prof, FMMLU_K_PANEL);
        frames_fut.get();
        Stage s2;
        s2.reserve_pinned(16 * 6 + sizeof(int) * (fslot.size() + fpos.size() + fbld.size()) +
                          sizeof(long long) * ftab.size());
        const size_t o_fs = s2.add(fslot), o_fp = s2.add(fpos), o_ft = s2.add(ftab), o_fb = s2.add(fbld);
        s2.upload(st);
        // Schur complement: Δ_{(S∪N)²} −= X_{(S∪N)R} · Up  (= X_{(S∪N)R} X_RR⁻¹ X_{R(S∪N)}), scattered
        // into the level BSR
        for (int w = 0; w < ph.nwaves(); ++w) {
        for (size_t e = ph.wrec[w]; e < (size_t)ph.wrec[w + 1]; ++e) {
          BoxJob& J = jobs[el[e]];
          BoxRec& R = recs[e];
          const int kn = R.k + J.nN;
          const FrameRef& fr = frames[e];
          GemmProblem P{};
          P.m = kn;
          P.n = kn;
          P.k = R.r;
          P.opA = kOpN;
          P.opB = kOpN;
          P.A = F + R.Lp;  // X_{(S∪N)R}
          P.lda = kn;
          P.B = F + R.Up;
          P.ldb = R.r;
          P.C = nullptr;
          P.ldc = 0;
          P.row0 = 0;
          P.col0 = sep ? kn : 0;
          P.ns = fr.ns;
          P.slot = s2.ptr<int>(o_fs) + fr.slot_off;
          P.pos = s2.ptr<int>(o_fp) + fr.slot_off;
          P.tab = s2.ptr<long long>(o_ft) + fr.tab_off;
          P.bld = s2.ptr<int>(o_fb) + fr.bld_off;
          add_gemm(gp, gt, P);
        }
        run_gemms(gp, gt, m1, 1, cur.bsr.as<cplx>(), st, keep, h->prof, FMMLU_K_SCHUR);
        }
        lap(21);
        // index arena + records
        h2d(ph.idx.p, hidx.data(), hidx.size() * sizeof(int), st);
        ph.recs.alloc(recs.size() * sizeof(BoxRec), st);
        h2d(ph.recs.p, recs.data(), recs.size() * sizeof(BoxRec), st);
        ph.nrec = (int)recs.size();
        ph.hrecs = recs;
        if (sep) {
          ph.recs_c.alloc(recsc.size() * sizeof(BoxRec), st);
          h2d(ph.recs_c.p, recsc.data(), recsc.size() * sizeof(BoxRec), st);
          ph.hrecs_c = recsc;
        }
        {
          std::vector<SolveItem> items;
          for (int w = 0; w < ph.nwaves(); ++w) {
            for (int e = ph.wrec[w]; e < ph.wrec[w + 1]; ++e)
              for (int c0 = 0; c0 < recs[e].k + recs[e].nN; c0 += kSolveChunk) items.push_back({e - ph.wrec[w], c0});
            ph.witem.push_back((int)items.size());
          }
          ph.nitems = (int)items.size();
          ph.items.alloc(std::max<size_t>(1, items.size()) * sizeof(SolveItem), st);
          if (!items.empty())
            h2d(ph.items.p, items.data(), items.size() * sizeof(SolveItem), st);
        }
        // no sync here: the next phase's ID preparation overlaps with this elimination on the GPU
        gmark(3);
        keep.push_back(std::move(s.dev));
        keep.push_back(std::move(s2.dev));
        track(h, -(long long)W.bytes);
        W.release();
        h->phases.push_back(std::move(ph));
      }
      if (prof_done) h->prof.resolve_first(prof_done);
      lap(4);
      track(h, -(long long)Tb.bytes);
      Tb.release();
      keep.clear();
      nextp = next_fut.get();
      lap(22);
    }
    lap(5);
    // carry state to the next (coarser) level
    for (int a = 0; a < no; ++a) {
      std::vector<int> na;
      for (int p : curpos[a]) na.push_back(cur.act[a][p]);
      act[cur.owners()[a]] = na;
      if (sep) {
        na.clear();
        for (int p : curposc[a]) na.push_back(cur.actc[a][p]);
        actc[cur.owners()[a]] = na;
      }
    }
    // Compact the level store to the still-active rows / columns (the skeletons; the eliminated R
    // rows and columns are never read again): the next level's build and the root read the compact
    // copy (workspace slot 1), and the big store (slot 0) is free for the next level.  cfg5: the
    // level-6 store shrinks from ≈ 45 GB to ≈ 9 GB, so two full level stores are never held at once.
    {
      std::vector<int> nactoff(no + 1, 0), fposr, fposc, pairoff(no + 1, 0);
      std::vector<long long> rowtot(no + 1, 0);
      for (int a = 0; a < no; ++a) {
        nactoff[a + 1] = nactoff[a] + (int)curpos[a].size();
        pairoff[a + 1] = pairoff[a] + (int)nb[a].size();
      }
      fposr.resize(nactoff[no]);
      if (sep) fposc.resize(nactoff[no]);
      HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {  // per owner: positions, block-row size
        for (int a = a0; a < a1; ++a) {
          std::copy(curpos[a].begin(), curpos[a].end(), fposr.begin() + nactoff[a]);
          if (sep) std::copy(curposc[a].begin(), curposc[a].end(), fposc.begin() + nactoff[a]);
          long long t = 0;
          for (int b : nb[a]) t += (long long)curpos[a].size() * curpos[b].size();
          rowtot[a + 1] = t;
        }
      });
      for (int a = 0; a < no; ++a) rowtot[a + 1] += rowtot[a];
      std::vector<long long> npoffv(pairoff[no]);
      const long long noff = rowtot[no];
      HostPool::get().parallel_for(no, 64, [&](int a0, int a1) {  // compact offsets of the owner's blocks
        for (int a = a0; a < a1; ++a) {
          long long o = rowtot[a];
          for (size_t i = 0; i < nb[a].size(); ++i) {
            npoffv[pairoff[a] + i] = o;
            cur.poff[a][i] = o;
            o += (long long)curpos[a].size() * curpos[nb[a][i]].size();
          }
        }
      });
      if (npoffv.empty()) npoffv.push_back(0);
      if (fposr.empty()) fposr.push_back(0);
      if (sep && fposc.empty()) fposc.push_back(0);
      Stage s;
      s.reserve_pinned(16 * 6 + sizeof(int) * (nactoff.size() + fposr.size() + fposc.size()) +
                       sizeof(long long) * npoffv.size());
      const size_t o_na = s.add(nactoff), o_np = s.add(npoffv), o_fr = s.add(fposr);
      const size_t o_fc = sep ? s.add(fposc) : o_fr;
      s.upload_owned(st);
      DBuf cbsr;
      borrow_ws(h, 1, cbsr, (size_t)std::max<long long>(noff, 1) * sizeof(cplx), st);
      int cid = h->prof.begin(FMMLU_K_BUILD, st);
      launch_compact_level(cur.npairs, cur.d_pair_a, cur.meta, s.ptr<int>(o_na), s.ptr<long long>(o_np),
                           s.ptr<int>(o_fr), s.ptr<int>(o_fc), cur.bsr.as<cplx>(), cbsr.as<cplx>(), st);
      h->prof.end(cid, st);
      h->prof.add(FMMLU_K_BUILD, 0.0, 32.0 * noff, 1);
      track(h, (long long)cbsr.bytes - (long long)cur.bsr.bytes);
      cur.bsr = std::move(cbsr);
      cur.size = noff;
      cur.meta.actoff = s.ptr<int>(o_na);
      cur.meta.poff = s.ptr<long long>(o_np);
      cur.meta_buf2 = std::move(s.dev);
      for (int a = 0; a < no; ++a) {  // the level's actives are now its final ones
        cur.act[a] = act[cur.owners()[a]];
        if (sep) cur.actc[a] = actc[cur.owners()[a]];
      }
    }
    std::fill(prevOwner.begin(), prevOwner.end(), -1);
    for (int a = 0; a < no; ++a) {
      for (size_t i = 0; i < cur.act[a].size(); ++i) {
        prevOwner[cur.act[a][i]] = a;
        prevPos[cur.act[a][i]] = (int)i;
      }
      if (sep)
        for (size_t i = 0; i < cur.actc[a].size(); ++i) {
          prevOwner[cur.actc[a][i]] = a;
          prevPosc[cur.actc[a][i]] = (int)i;
        }
    }
    prev = std::move(cur);
    S.t_levels_ms[lvl] = now_ms() - tl0;  // host-side span of the level (GPU work may still drain)
    if (trace) {  // host-time sections of this level (same order as the summary line at the end)
      static double trp[24];
      if (lvl == L - 1) std::memset(trp, 0, sizeof(trp));
      fprintf(stderr, "[fmmlu] L%d host ms by section:", lvl);
      for (int i = 0; i < 23; ++i) {
        if (tr[i] - trp[i] > 0.05) fprintf(stderr, " s%d %.1f", i, tr[i] - trp[i]);
        trp[i] = tr[i];
      }
      fprintf(stderr, " | span %.1f\n", S.t_levels_ms[lvl]);
    }
  }

  lap(6);
  if (trace) {
    fprintf(stderr, "[fmmlu] allocator host ms: cudaMallocAsync %.1f (%lld calls, max %.1f) cudaFreeAsync %.1f "
                    "cudaMallocHost %.1f\n",
            g_ac.alloc_ms, g_ac.nalloc, g_ac.alloc_max, g_ac.free_ms, g_ac.pin_ms);
    g_ac = AllocClock{};
  }
  if (trace)
    fprintf(stderr, "[fmmlu] host ms: level-setup %.1f build-tasks %.1f phase-jobs %.1f id %.1f elim %.1f "
                    "update %.1f carry %.1f other %.1f | id: tasks %.1f gatherlaunch %.1f gram %.1f prep %.1f "
                    "pchol %.1f rest %.1f | topo %.1f acts %.1f | elim: sizes %.1f alloc %.1f tasks %.1f "
                    "upload %.1f EF %.1f inv-panel-schur+recs %.1f | next-prep wait %.1f | wait %.1f\n",
            tr[0], tr[1], tr[2], tr[3], tr[4], tr[5], tr[6], tr[7], tr[8], tr[9], tr[10], tr[11], tr[12], tr[13],
            tr[14], tr[15], tr[16], tr[17], tr[18], tr[19], tr[20], tr[21], tr[22], S.t_sync_wait_ms);
  // ------------------------------------------------------------------ root
  gmark(4);
  double tr0 = now_ms();
  std::vector<int> Bt;
  if (prev.level >= 0) {
    for (size_t a = 0; a < prev.owners().size(); ++a)
      for (int g : act[prev.owners()[a]]) Bt.push_back(g);
  } else {
    for (int i = 0; i < n; ++i) Bt.push_back(i);
  }
  std::sort(Bt.begin(), Bt.end());
  std::vector<int> Btc_store;  // separate IDs: the root's columns B_t^c (as many as its rows)
  if (sep) {
    if (prev.level >= 0) {
      for (size_t a = 0; a < prev.owners().size(); ++a)
        for (int g : actc[prev.owners()[a]]) Btc_store.push_back(g);
    } else {
      Btc_store = Bt;
    }
    std::sort(Btc_store.begin(), Btc_store.end());
  }
  const std::vector<int>& Btc = sep ? Btc_store : Bt;
  const int n0 = (int)Bt.size();
  h->n0 = n0;
  {
    // The idle shared-workspace slots (M, T, W, Gram, and the level store the root does not read)
    // are kept for the next factorization unless the root block would not fit beside them: cfg5
    // holds ≈ 120 GB of workspace + 45 GB of factors at this point.
    size_t fr = 0, tot = 0;
    FMMLU_CUDA(cudaMemGetInfo(&fr, &tot));
    uint64_t res = 0, used = 0;
    cudaMemPool_t pool = lib_pool(h->dev);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    const size_t avail = fr + (size_t)(res - used) + big_cache(h->dev).cached();
    const size_t need = (size_t)n0 * n0 * sizeof(cplx) * 2 + (4ull << 30);
    if (avail < need) {
      const int keep_slot = prev.level >= 0 ? 1 : -1;  // the compacted store the root reads
      for (int sl = 0; sl < 6; ++sl)
        if (sl != keep_slot && h->ws[sl].p) {
          h->ws[sl].st = st;
          h->ws[sl].release();
        }
      big_cache(h->dev).flush(st);
    }
  }
  S.n0 = n0;
  if (n0 > 0) {
    h->root.alloc((size_t)n0 * n0 * sizeof(cplx), st);
    track(h, h->root.bytes);
    S.factor_bytes += h->root.bytes;
    std::vector<int> slot(n0), pos(n0), bld;
    std::vector<int> slotc(sep ? n0 : 0), posc(sep ? n0 : 0);
    std::vector<long long> tab;
    int ns = 1;
    if (prev.level >= 0) {
      ns = (int)prev.owners().size();
      for (int i = 0; i < n0; ++i) {
        slot[i] = prevOwner[Bt[i]];
        pos[i] = prevPos[Bt[i]];
      }
      if (sep)
        for (int i = 0; i < n0; ++i) {
          slotc[i] = prevOwner[Btc[i]];
          posc[i] = prevPosc[Btc[i]];
        }
      tab.assign((size_t)ns * ns, -1);
      for (int a = 0; a < ns; ++a)
        for (int b = 0; b < ns; ++b) tab[(size_t)a * ns + b] = prev.off(a, b);
      for (int a = 0; a < ns; ++a) bld.push_back((int)prev.act[a].size());
    } else {
      std::fill(slot.begin(), slot.end(), -1);
      std::fill(slotc.begin(), slotc.end(), -1);
      tab.push_back(-1);
      bld.push_back(0);
    }
    std::vector<BuildTask> tasks;
    for (int i0 = 0; i0 < n0; i0 += kTile)
      for (int j0 = 0; j0 < n0; j0 += kTile) {
        BuildTask t{};
        t.dst = 0;
        t.ldd = n0;
        t.rows_off = 0;
        t.cols_off = 0;
        t.i0 = i0;
        t.j0 = j0;
        t.ni = std::min(kTile, n0 - i0);
        t.nj = std::min(kTile, n0 - j0);
        t.ns = ns;
        t.tab_off = 0;
        t.bld_off = 0;
        tasks.push_back(t);
      }
    Stage s;
    size_t o_t = s.add(tasks), o_g = s.add(Bt), o_s = s.add(slot), o_p = s.add(pos), o_tab = s.add(tab),
           o_b = s.add(bld);
    const size_t o_gc = sep ? s.add(Btc) : o_g, o_sc = sep ? s.add(slotc) : o_s, o_pc = sep ? s.add(posc) : o_p;
    s.upload(st);
    int rid = h->prof.begin(FMMLU_K_ROOT, st);
    launch_build(s.ptr<BuildTask>(o_t), (int)tasks.size(), s.ptr<int>(o_g), s.ptr<int>(o_s), s.ptr<int>(o_p),
                 s.ptr<long long>(o_tab), s.ptr<int>(o_b), prev.bsr.as<cplx>(), h->root.as<cplx>(), h->g, k, st,
                 s.ptr<int>(o_gc), s.ptr<int>(o_sc), s.ptr<int>(o_pc));
    h->prof.end(rid, st);
    h->prof.add(FMMLU_K_ROOT, 60.0 * (double)n0 * n0, 16.0 * (double)n0 * n0, 1);
    // dense LU with partial pivoting of the root block
    std::vector<DBuf> rkeep;
    DBuf piv;
    piv.alloc((size_t)n0 * sizeof(int), st);
    const int TB = root_lu_tb(n0), nblk = (n0 + TB - 1) / TB;
    h->root_dinv.alloc((size_t)2 * nblk * TB * TB * sizeof(cplx), st);
    h->root_flags.alloc((size_t)2 * (nblk + 1) * sizeof(int), st);
    track(h, h->root_dinv.bytes);
    S.factor_bytes += h->root_dinv.bytes;
    const cplx m1 = cmk(-1.0, 0.0);
    int lid = h->prof.begin(FMMLU_K_ROOT, st);
    {
      static const bool lookahead = !(getenv("FMMLU_ROOT_LOOKAHEAD") && atoi(getenv("FMMLU_ROOT_LOOKAHEAD")) == 0);
      cudaStream_t sp = st;
      if (lookahead) FMMLU_CUDA(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
      struct SideStream {  // its staging arena is dropped and the stream destroyed on every path
        cudaStream_t s, main;
        ~SideStream() {
          if (s != main) {
            cudaStreamSynchronize(s);
            drop_arena(s);
            cudaStreamDestroy(s);
          }
        }
      } side{sp, st};
      root_lu_factor(h->root.as<cplx>(), n0, piv.as<int>(), status.as<int>(), h->root_dinv.as<cplx>(), st, sp,
                     [&](cudaStream_t gs, int m, int nn, int kk, const cplx* A, int lda, const cplx* B, int ldb, cplx* C,
                         int ldc) {
                       std::vector<GemmProblem> gp;
                       std::vector<GemmGroup> gt;
                       GemmProblem P{};
                       P.m = m;
                       P.n = nn;
                       P.k = kk;
                       P.opA = kOpN;
                       P.opB = kOpN;
                       P.A = A;
                       P.lda = lda;
                       P.B = B;
                       P.ldb = ldb;
                       P.C = C;
                       P.ldc = ldc;
                       add_gemm(gp, gt, P);
                       gemm_batched_staged(gp, gt, m1, gs, rkeep);
                     });
      // the staging buffers of the side stream (rkeep entries borrowed from its arena) end with it
      FMMLU_CUDA(cudaStreamSynchronize(sp));
    }
    h->prof.end(lid, st);
    h->prof.add(FMMLU_K_ROOT, 8.0 / 3.0 * (double)n0 * n0 * n0, 32.0 * (double)n0 * n0, root_lu_launches(n0));
    int* hp = h->d2h(n0);
    FMMLU_CUDA(cudaMemcpyAsync(hp, piv.p, (size_t)n0 * sizeof(int), cudaMemcpyDeviceToHost, st));
    wait_stream(h, st);
    // σ = the interchanges composed in order (P·y)[i] = y[σ(i)]; rows_in = B_t∘σ
    std::vector<int> sig(n0), rin(n0);
    for (int i = 0; i < n0; ++i) sig[i] = i;
    for (int j = 0; j < n0; ++j) std::swap(sig[j], sig[hp[j]]);
    for (int i = 0; i < n0; ++i) rin[i] = Bt[sig[i]];
    h->root_rows.alloc((size_t)n0 * sizeof(int), st);
    h->root_rows_in.alloc((size_t)n0 * sizeof(int), st);
    h2d(h->root_rows.p, Btc.data(), n0 * sizeof(int), st);  // the solve writes the unknowns at B_t^c
    h2d(h->root_rows_in.p, rin.data(), n0 * sizeof(int), st);
    wait_stream(h, st);
  }
  if (sep) {
    if ((int)Btc.size() != n0) throw Error(FMMLU_ECUDA, "separate IDs: root rows / columns differ in number");
    // a bijection: the root's unknowns pair with its equations (both sweeps overwrite those entries)
    for (int i = 0; i < n0; ++i) sep_pi[Btc[i]] = Bt[i];
    h->sep_perm.alloc((size_t)std::max(n, 1) * sizeof(int), st);
    h2d(h->sep_perm.p, sep_pi.data(), (size_t)n * sizeof(int), st);
    wait_stream(h, st);
  }
  if (prev.bsr.p) track(h, -(long long)prev.bsr.bytes);
  prev.bsr.release();
  // the shared workspace stays allocated for the next factorization on this device; the stream was
  // synchronised above, so the next user (on any stream) may reuse it at once
  int hstatus = 0;
  FMMLU_CUDA(cudaMemcpyAsync(&hstatus, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  wait_stream(h, st);
  h->prof.resolve();
  S.t_root_ms = now_ms() - tr0;
  if (trace && !gmarks.empty()) {
    gmark(5);
    FMMLU_CUDA(cudaStreamSynchronize(st));
    static const char* nm[6] = {"id_begin", "id_end", "el_begin", "el_end", "root_begin", "end"};
    std::map<std::pair<int, int>, std::pair<double, int>> agg;
    for (size_t i = 0; i + 1 < gmarks.size(); ++i) {
      float ms = 0.f;
      FMMLU_CUDA(cudaEventElapsedTime(&ms, gmarks[i].second, gmarks[i + 1].second));
      auto& a = agg[{gmarks[i].first, gmarks[i + 1].first}];
      a.first += ms;
      a.second += 1;
    }
    float tot = 0.f;
    FMMLU_CUDA(cudaEventElapsedTime(&tot, gmarks.front().second, gmarks.back().second));
    fprintf(stderr, "[fmmlu] device timeline (%.2f ms from the first ID to the end):", tot);
    for (auto& kv : agg)
      fprintf(stderr, " %s->%s %.2f ms (%d)", nm[kv.first.first], nm[kv.first.second], kv.second.first, kv.second.second);
    fprintf(stderr, "\n");
    for (auto& m : gmarks) cudaEventDestroy(m.second);
  }
  if (hstatus) throw Error(FMMLU_ESINGULAR, "exactly singular pivot block (X_RR or root)");
  h->k = k;
  h->eps = eps;
  h->factored = true;
}

// ---- multi-RHS sweeps on the DMMA GEMM (the same operators as the
// per-box kernels below): y (tree order, W^{½}-scaled, ld ldy) ← Ã⁻¹ y for
// Q columns.  Per phase the boxes' rows are gathered into dense blocks, the products run as
// batched GEMMs (C += α op(A) B), and the results are scattered back (atomics on shared N rows).
// nrhs from which the GEMM sweeps replace the per-box kernels (FMMLU_GEMM_SOLVE_MIN overrides)
const int kGemmSolveMin = getenv("FMMLU_GEMM_SOLVE_MIN") ? std::max(1, atoi(getenv("FMMLU_GEMM_SOLVE_MIN"))) : 32;

void sweeps_gemm(fmmlu_handle* h, cplx* y, int ldy, int Q) {
  cudaStream_t st = h->stream;
  Prof& P = h->prof;
  std::vector<DBuf> keep;
  std::vector<GemmProblem> gp;
  std::vector<GemmGroup> gt;
  const cplx m1 = cmk(-1.0, 0.0), p1 = cmk(1.0, 0.0);
  size_t wsmax = 1;
  for (auto& ph : h->phases) {
    size_t w = 0;
    for (auto& R : ph.hrecs) w += (size_t)(2 * (R.k + R.nN) + 2 * R.r) * Q;
    wsmax = std::max(wsmax, w);
  }
  DBuf ws;
  ws.alloc(wsmax * sizeof(cplx), st);
  cplx* W = ws.as<cplx>();
  // per phase: gathered blocks (YSN, YR of every box) first, then the accumulators (Z, DSN)
  // in one contiguous region [z0, tot) that a single memset clears
  auto layout = [&](const Phase& ph, std::vector<SweepWs>& L, long long& z0) {
    long long o = 0;
    L.resize(ph.hrecs.size());
    for (size_t e = 0; e < ph.hrecs.size(); ++e) {
      const BoxRec& R = ph.hrecs[e];
      L[e].ysn = o;
      o += (long long)(R.k + R.nN) * Q;
      L[e].yr = o;
      o += (long long)R.r * Q;
    }
    z0 = o;
    for (size_t e = 0; e < ph.hrecs.size(); ++e) {
      const BoxRec& R = ph.hrecs[e];
      L[e].z = o;
      o += (long long)R.r * Q;
      L[e].dsn = o;
      o += (long long)(R.k + R.nN) * Q;
    }
    return o;
  };
  auto prob = [&](int m, int n, int k, int opA, const cplx* A, int lda, const cplx* B, int ldb, cplx* C, int ldc) {
    GemmProblem g{};
    g.m = m;
    g.n = n;
    g.k = k;
    g.opA = opA;
    g.opB = kOpN;
    g.A = A;
    g.lda = std::max(lda, 1);
    g.B = B;
    g.ldb = std::max(ldb, 1);
    g.C = C;
    g.ldc = std::max(ldc, 1);
    add_gemm(gp, gt, g);
  };
  const int id = P.begin(FMMLU_K_SOLVE, st);
  // ---- upward: E (t = y_R − Tᵀ y_S), then Lp t and X_RR⁻¹ t
  for (auto& ph : h->phases) {
    if (ph.nrec <= 0) continue;
    std::vector<SweepWs> L;
    long long z0 = 0;
    const long long tot = layout(ph, L, z0);
    Stage s;
    const size_t oL = s.add(L);
    s.upload(st);
    const SweepWs* dL = s.ptr<SweepWs>(oL);
    const cplx* F = ph.fac.as<cplx>();
    FMMLU_CUDA(cudaMemsetAsync(W + z0, 0, (size_t)(tot - z0) * sizeof(cplx), st));
    launch_sweep_move(ph.recs.as<BoxRec>(), dL, ph.nrec, ph.idx.as<int>(), y, ldy, Q, W, 0, st);
    for (size_t e = 0; e < L.size(); ++e) {
      const BoxRec& R = ph.hrecs[e];
      if (R.k > 0) prob(R.r, Q, R.k, kOpT, F + R.T, R.k, W + L[e].ysn, R.k + R.nN, W + L[e].yr, R.r);
    }
    run_gemms(gp, gt, m1, 0, nullptr, st, keep, P, FMMLU_K_SOLVE);
    for (size_t e = 0; e < L.size(); ++e) {  // z = X_RR⁻¹ t
      const BoxRec& R = ph.hrecs[e];
      prob(R.r, Q, R.r, kOpN, F + R.Xi, R.r, W + L[e].yr, R.r, W + L[e].z, R.r);
    }
    run_gemms(gp, gt, p1, 0, nullptr, st, keep, P, FMMLU_K_SOLVE);
    for (size_t e = 0; e < L.size(); ++e) {  // X_{(S∪N)R} z  (= Lp t)
      const BoxRec& R = ph.hrecs[e];
      const int kn = R.k + R.nN;
      prob(kn, Q, R.r, kOpN, F + R.Lp, kn, W + L[e].z, R.r, W + L[e].dsn, kn);
    }
    run_gemms(gp, gt, p1, 0, nullptr, st, keep, P, FMMLU_K_SOLVE);
    for (int w = 0; w < ph.nwaves(); ++w)
      launch_sweep_move(ph.recs.as<BoxRec>() + ph.wrec[w], dL + ph.wrec[w], ph.wrec[w + 1] - ph.wrec[w],
                        ph.idx.as<int>(), y, ldy, Q, W, 1, st);
    keep.push_back(std::move(s.dev));
  }
  // ---- root: y[B_t] ← A_t⁻¹ y[B_t] (LU triangular solves)
  SepSwap swp;
  cplx* const yeq = y;  // the equation-side vector
  if (cplx* y2 = swp.begin(h, y, ldy, Q, st)) y = y2;
  if (h->n0 > 0) {
    int rid = P.begin(FMMLU_K_SOLVE, st);
    root_solve(h, yeq, ldy, Q, st, y);
    P.end(rid, st);
    P.add(FMMLU_K_SOLVE, 8.0 * (double)h->n0 * h->n0 * Q, 16.0 * (double)h->n0 * h->n0, 4);
  }
  // ---- downward (reverse order): U (y_R −= Up y_{S∪N}), then F (y_S −= T y_R)
  for (auto it = h->phases.rbegin(); it != h->phases.rend(); ++it) {
    Phase& ph = *it;
    if (ph.nrec <= 0) continue;
    std::vector<SweepWs> L;
    long long z0 = 0;
    const long long tot = layout(ph, L, z0);
    Stage s;
    const size_t oL = s.add(L);
    s.upload(st);
    const SweepWs* dL = s.ptr<SweepWs>(oL);
    const cplx* F = ph.fac.as<cplx>();
    FMMLU_CUDA(cudaMemsetAsync(W + z0, 0, (size_t)(tot - z0) * sizeof(cplx), st));
    launch_sweep_move(ph.down_recs(), dL, ph.nrec, ph.idx.as<int>(), y, ldy, Q, W, 0, st);
    for (size_t e = 0; e < L.size(); ++e) {
      const BoxRec& R = ph.down_hrecs()[e];
      const int kn = R.k + R.nN;
      prob(R.r, Q, kn, kOpN, F + R.Up, R.r, W + L[e].ysn, kn, W + L[e].yr, R.r);
    }
    run_gemms(gp, gt, m1, 0, nullptr, st, keep, P, FMMLU_K_SOLVE);
    for (size_t e = 0; e < L.size(); ++e) {
      const BoxRec& R = ph.down_hrecs()[e];
      if (R.k > 0) prob(R.k, Q, R.r, kOpN, F + R.T, R.k, W + L[e].yr, R.r, W + L[e].dsn, R.k);
    }
    run_gemms(gp, gt, p1, 0, nullptr, st, keep, P, FMMLU_K_SOLVE);
    for (int w = 0; w < ph.nwaves(); ++w)
      launch_sweep_move(ph.down_recs() + ph.wrec[w], dL + ph.wrec[w], ph.wrec[w + 1] - ph.wrec[w],
                        ph.idx.as<int>(), y, ldy, Q, W, 2, st);
    keep.push_back(std::move(s.dev));
  }
  swp.end(h, yeq, Q, st);
  P.end(id, st);
  wait_stream(h, st);  // keep (staging, workspace) outlives the launches; resets the staging arenas
}

// GEMM sweeps or per-box kernels?  Deterministic mode and ≥ 32 RHS: GEMM sweeps.  Between 16 and 31 RHS
// the crossover depends on the size of the factor store (measured, tools/solve_scan.py: cfg5 with 44.7 GB
// of factors 113 vs 132 ms at 16 RHS and 160 vs 252 ms at 31 in favour of the GEMM sweeps; cfg3 with
// 4.3 GB 35 vs 22 ms at 16 RHS in favour of the per-box kernels): GEMM sweeps from 16 RHS for stores
// of ≥ 16 GB.  FMMLU_GEMM_SOLVE_MIN overrides both thresholds.
bool use_gemm_sweeps(const fmmlu_handle* h, int nrhs) {
  static const bool forced = getenv("FMMLU_GEMM_SOLVE_MIN") != nullptr;
  if (is_deterministic(h) || nrhs >= kGemmSolveMin) return true;
  return !forced && nrhs >= 16 && h->stats.factor_bytes >= (16ll << 30);
}

// RHS columns per GEMM-sweep pass: bounded so the phase workspace stays ≤ ~2 GB
int sweep_chunk(const fmmlu_handle* h, int nrhs) {
  size_t per = 1;
  for (auto& ph : h->phases) {
    size_t w = 0;
    for (auto& R : ph.hrecs) w += (size_t)(2 * (R.k + R.nN) + 2 * R.r);
    per = std::max(per, w);
  }
  const size_t cap = (size_t)2e9 / (per * sizeof(cplx));
  return (int)std::max<size_t>(kGemmSolveMin, std::min<size_t>({(size_t)nrhs, cap, (size_t)1024}));
}

// The per-box solve sweeps: V⁻¹ phase by phase, the root, W⁻¹ in reverse; each
// phase's kernels run once per sub-wave (one wave unless deterministic).  scr: Σr × nrhs scratch.
void sweeps_boxes(fmmlu_handle* h, cplx* y, int ldy, int nrhs, cplx* scr, cudaStream_t st, cplx* root_tmp = nullptr) {
  static const bool trace_env = getenv("FMMLU_TRACE") != nullptr;
  const bool trace = trace_env && root_tmp == nullptr;  // (no event queries inside a stream capture)
  cudaEvent_t ev[4];
  if (trace)
    for (auto& e : ev) FMMLU_CUDA(cudaEventCreate(&e));
  if (trace) FMMLU_CUDA(cudaEventRecord(ev[0], st));
  for (auto& ph : h->phases)
    for (int w = 0; w < ph.nwaves(); ++w)
      launch_solve_up2(ph.recs.as<BoxRec>() + ph.wrec[w], ph.wrec[w + 1] - ph.wrec[w],
                       ph.items.as<SolveItem>() + ph.witem[w], ph.witem[w + 1] - ph.witem[w], ph.fac.as<cplx>(),
                       ph.idx.as<int>(), y, ldy, nrhs, scr, st, ph.kmax, ph.rmax);
  if (trace) FMMLU_CUDA(cudaEventRecord(ev[1], st));
  SepSwap swp;
  cplx* const yeq = y;
  if (cplx* y2 = swp.begin(h, y, ldy, nrhs, st)) y = y2;
  root_solve(h, yeq, ldy, nrhs, st, y, root_tmp);
  if (trace) FMMLU_CUDA(cudaEventRecord(ev[2], st));
  for (auto it = h->phases.rbegin(); it != h->phases.rend(); ++it) {
    FMMLU_CUDA(cudaMemsetAsync(scr, 0, (size_t)it->tmp_rows * nrhs * sizeof(cplx), st));
    for (int w = it->nwaves() - 1; w >= 0; --w)
      launch_solve_down2(it->down_recs() + it->wrec[w], it->wrec[w + 1] - it->wrec[w],
                         it->items.as<SolveItem>() + it->witem[w], it->witem[w + 1] - it->witem[w],
                         it->fac.as<cplx>(), it->idx.as<int>(), y, ldy, nrhs, scr, st, it->rmax, it->kmax);
  }
  swp.end(h, yeq, nrhs, st);
  if (trace) {
    FMMLU_CUDA(cudaEventRecord(ev[3], st));
    FMMLU_CUDA(cudaEventSynchronize(ev[3]));
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    fprintf(stderr, "[fmmlu] solve (%d RHS, per-box kernels): up %.3f ms, root %.3f ms (n0 %lld), down %.3f ms\n", nrhs,
            a, b, (long long)h->n0, c);
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void solve_impl(fmmlu_handle* h, void* rhs, int nrhs) {
  cudaStream_t st = h->stream;
  const int n = (int)h->n;
  const bool dev = is_device_ptr(rhs);
  DBuf io, y;
  cplx* b = reinterpret_cast<cplx*>(rhs);
  if (!dev) {
    io.alloc((size_t)n * nrhs * sizeof(cplx), st);
    FMMLU_CUDA(cudaMemcpyAsync(io.p, rhs, (size_t)n * nrhs * sizeof(cplx), cudaMemcpyHostToDevice, st));
    b = io.as<cplx>();
  }
  // Small-RHS solves from the second call with the same nrhs on: one CUDA graph (see SolveGraph).
  static const bool graph_env = !(getenv("FMMLU_SOLVE_GRAPH") && atoi(getenv("FMMLU_SOLVE_GRAPH")) == 0);
  static const bool trace_env = getenv("FMMLU_TRACE") != nullptr;
  const bool gemm_path = use_gemm_sweeps(h, nrhs);
  const bool graph_ok = graph_env && !trace_env && !gemm_path && !h->fac_separate;
  size_t scr_rows = 1;
  for (auto& ph : h->phases) scr_rows = std::max(scr_rows, (size_t)ph.tmp_rows);
  DBuf scr;
  cplx* yp = nullptr;
  cplx* scrp = nullptr;
  cplx* rootp = nullptr;
  if (graph_ok) {  // persistent buffers: the graphs hold their addresses
    const size_t ny = (size_t)n * nrhs * sizeof(cplx), ns = scr_rows * nrhs * sizeof(cplx),
                 nr = (size_t)std::max<long long>(h->n0, 1) * nrhs * sizeof(cplx);
    if (h->sv_y.bytes < ny || h->sv_scr.bytes < ns || h->sv_root.bytes < nr) {
      h->drop_solve_graphs();
      if (h->sv_y.bytes < ny) h->sv_y.alloc(ny, st);
      if (h->sv_scr.bytes < ns) h->sv_scr.alloc(ns, st);
      if (h->sv_root.bytes < nr) h->sv_root.alloc(nr, st);
    }
    yp = h->sv_y.as<cplx>();
    scrp = h->sv_scr.as<cplx>();
    rootp = h->sv_root.as<cplx>();
  } else {
    y.alloc((size_t)n * nrhs * sizeof(cplx), st);
    yp = y.as<cplx>();
  }
  Prof& P = h->prof;
  int sid = P.begin(FMMLU_K_SOLVE, st);
  launch_permute_in(b, n, yp, n, nrhs, h->perm.as<long long>(), h->g.sw, 1, st);
  // many right-hand sides: the sweeps as batched DMMA GEMMs; also the deterministic path (the
  // per-box kernels split a box's product over CTAs that meet in fp64 atomics)
  if (gemm_path) {
    P.end(sid, st);
    const int qc = sweep_chunk(h, nrhs);
    for (int q0 = 0; q0 < nrhs; q0 += qc) sweeps_gemm(h, yp + (size_t)q0 * n, n, std::min(qc, nrhs - q0));
    sid = P.begin(FMMLU_K_SOLVE, st);
    launch_permute_out(yp, b, n, n, nrhs, h->perm.as<long long>(), h->g.sw, 1, st);
    P.end(sid, st);
    if (!dev)
      FMMLU_CUDA(cudaMemcpyAsync(rhs, io.p, (size_t)n * nrhs * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    FMMLU_CUDA(cudaStreamSynchronize(st));
    P.resolve();
    return;
  }
  if (graph_ok) {
    fmmlu_handle::SolveGraph& G = h->solve_graphs[nrhs];
    if (!G.exec && G.uses >= 1) {  // second solve with this nrhs: capture the sweeps
      cudaGraph_t graph = nullptr;
      FMMLU_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        sweeps_boxes(h, yp, n, nrhs, scrp, st, rootp);
      } catch (...) {
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      FMMLU_CUDA(cudaStreamEndCapture(st, &graph));
      const cudaError_t ie = cudaGraphInstantiate(&G.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        G.exec = nullptr;
        FMMLU_CUDA(ie);
      }
    }
    if (G.exec) FMMLU_CUDA(cudaGraphLaunch(G.exec, st));
    else sweeps_boxes(h, yp, n, nrhs, scrp, st, rootp);
    ++G.uses;
  } else {
    scr.alloc(scr_rows * nrhs * sizeof(cplx), st);
    sweeps_boxes(h, yp, n, nrhs, scr.as<cplx>(), st);
  }
  launch_permute_out(yp, b, n, n, nrhs, h->perm.as<long long>(), h->g.sw, 1, st);
  P.end(sid, st);
  {
    // algorithmic: every stored factor entry read once, 8 flops per entry per RHS
    double entries = (double)h->n0 * h->n0;
    for (auto& ph : h->phases) entries += (double)ph.fac_bytes / 16.0;
    P.add(FMMLU_K_SOLVE, 8.0 * entries * nrhs, 16.0 * entries + 64.0 * n * nrhs,
          2 + 6 * (long long)h->phases.size() + (h->n0 > 0 ? 3 : 0));
  }
  if (!dev)
    FMMLU_CUDA(cudaMemcpyAsync(rhs, io.p, (size_t)n * nrhs * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  FMMLU_CUDA(cudaStreamSynchronize(st));
  P.resolve();
}

// ---- forward factored apply
// A ≈ V₁⋯V_M P_t D P_tᵀ W_M⋯W₁ with D = diag(X_{R_jR_j}, A_{B_tB_t}).  The factor store keeps
// X_RR⁻¹ and X_t⁻¹ (reading R3); their inverses are formed once, on the first apply, by the same
// batched Gauss-Jordan kernels and cached until the next factorization.
void apply_prepare(fmmlu_handle* h) {
  cudaStream_t st = h->stream;
  DBuf status;
  status.alloc(16, st);
  FMMLU_CUDA(cudaMemsetAsync(status.p, 0, 16, st));
  std::vector<DBuf> keep;
  for (auto& ph : h->phases) {
    if (ph.nrec <= 0) continue;
    std::vector<BoxRec> recs(ph.nrec);  // separate IDs: D acts on the unknowns at R_c (column records)
    FMMLU_CUDA(cudaMemcpyAsync(recs.data(), ph.down_recs(), recs.size() * sizeof(BoxRec), cudaMemcpyDeviceToHost, st));
    FMMLU_CUDA(cudaStreamSynchronize(st));
    long long off = 0;
    std::vector<std::pair<long long, int>> mats;
    for (auto& R : recs) {
      R.Xi = off;
      mats.push_back({off, R.r});
      off += (long long)R.r * R.r;
    }
    ph.ap_xs.alloc(std::max<long long>(1, off) * sizeof(cplx), st);
    ph.ap_recs.alloc(recs.size() * sizeof(BoxRec), st);
    FMMLU_CUDA(cudaMemcpyAsync(ph.ap_recs.p, recs.data(), recs.size() * sizeof(BoxRec), cudaMemcpyHostToDevice, st));
    track(h, ph.ap_xs.bytes);
    launch_apply_copyX(ph.recs.as<BoxRec>(), ph.ap_recs.as<BoxRec>(), ph.nrec, ph.fac.as<cplx>(),
                       ph.ap_xs.as<cplx>(), st);
    std::vector<std::pair<cplx*, int>> mp;
    for (auto& m : mats)
      if (m.second > 0) mp.push_back({ph.ap_xs.as<cplx>() + m.first, m.second});
    gj_blocked(h, mp, status.as<int>(), keep, FMMLU_K_APPLY);
    FMMLU_CUDA(cudaStreamSynchronize(st));  // recs (host) and the staging arena are reused next phase
    keep.clear();
  }
  int hstatus = 0;
  FMMLU_CUDA(cudaMemcpyAsync(&hstatus, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  wait_stream(h, st);
  h->prof.resolve();
  if (hstatus) throw Error(FMMLU_ESINGULAR, "singular stored inverse while preparing fmmlu_apply");
  h->apply_ready = true;
}

void apply_impl(fmmlu_handle* h, void* xio, int nrhs) {
  cudaStream_t st = h->stream;
  if (!h->apply_ready) apply_prepare(h);
  const int n = (int)h->n;
  const bool dev = is_device_ptr(xio);
  DBuf io, y;
  cplx* b = reinterpret_cast<cplx*>(xio);
  if (!dev) {
    io.alloc((size_t)n * nrhs * sizeof(cplx), st);
    FMMLU_CUDA(cudaMemcpyAsync(io.p, xio, (size_t)n * nrhs * sizeof(cplx), cudaMemcpyHostToDevice, st));
    b = io.as<cplx>();
  }
  y.alloc((size_t)n * nrhs * sizeof(cplx), st);
  cplx* yp = y.as<cplx>();
  Prof& P = h->prof;
  int sid = P.begin(FMMLU_K_APPLY, st);
  launch_permute_in(b, n, yp, n, nrhs, h->perm.as<long long>(), h->g.sw, 1, st);  // W^{½} x, tree order
  size_t scr_rows = 1;
  for (auto& ph : h->phases) scr_rows = std::max(scr_rows, (size_t)ph.tmp_rows);
  DBuf scr;
  scr.alloc(scr_rows * nrhs * sizeof(cplx), st);
  for (auto& ph : h->phases) {  // W_M⋯W₁ x: W₁ first
    FMMLU_CUDA(cudaMemsetAsync(scr.p, 0, (size_t)ph.tmp_rows * nrhs * sizeof(cplx), st));
    for (int w = 0; w < ph.nwaves(); ++w)
      launch_apply_w(ph.down_recs() + ph.wrec[w], ph.wrec[w + 1] - ph.wrec[w],
                     ph.items.as<SolveItem>() + ph.witem[w], ph.witem[w + 1] - ph.witem[w], ph.fac.as<cplx>(),
                     ph.idx.as<int>(), yp, n, nrhs, scr.as<cplx>(), st, ph.rmax, ph.kmax);
  }
  for (auto& ph : h->phases)  // D on the R blocks
    launch_apply_d(ph.ap_recs.as<BoxRec>(), ph.nrec, ph.ap_xs.as<cplx>(), ph.idx.as<int>(), yp, n, nrhs,
                   scr.as<cplx>(), st, ph.rmax);
  // separate IDs: D mapped the unknowns at R_c in place; the products belong to the equations R_r,
  // y2[sep_perm[c]] = y[c], and the root block maps y[B_t^c] to y2[B_t]; the V sweep runs on y2
  DBuf y2;
  if (h->fac_separate) {
    y2.alloc((size_t)n * nrhs * sizeof(cplx), st);
    launch_rows_move(h->sep_perm.as<int>(), n, y2.as<cplx>(), n, yp, nrhs, 1, st);
    root_fwd(h, yp, n, nrhs, st, y2.as<cplx>());
    yp = y2.as<cplx>();
  } else {
    root_fwd(h, yp, n, nrhs, st);  // P_t A_{B_tB_t} P_tᵀ from the stored L·U
  }
  for (auto it = h->phases.rbegin(); it != h->phases.rend(); ++it)  // V₁⋯V_M: V_M first
    for (int w = it->nwaves() - 1; w >= 0; --w)
      launch_apply_v(it->recs.as<BoxRec>() + it->wrec[w], it->wrec[w + 1] - it->wrec[w],
                     it->items.as<SolveItem>() + it->witem[w], it->witem[w + 1] - it->witem[w], it->fac.as<cplx>(),
                     it->idx.as<int>(), yp, n, nrhs, scr.as<cplx>(), st, it->rmax);
  launch_permute_out(yp, b, n, n, nrhs, h->perm.as<long long>(), h->g.sw, 1, st);  // W^{-½}, caller order
  P.end(sid, st);
  {
    double entries = 2.0 * (double)h->n0 * h->n0;
    for (auto& ph : h->phases) entries += (double)ph.fac_bytes / 16.0;
    P.add(FMMLU_K_APPLY, 8.0 * entries * nrhs, 16.0 * entries + 64.0 * n * nrhs,
          2 + 8 * (long long)h->phases.size() + (h->n0 > 0 ? 3 : 0));
  }
  if (!dev)
    FMMLU_CUDA(cudaMemcpyAsync(xio, io.p, (size_t)n * nrhs * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  FMMLU_CUDA(cudaStreamSynchronize(st));
  P.resolve();
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FMMLU_OK;
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(FMMLU_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(FMMLU_ECUDA, e.what());
  }
}

void tune_malloc() {  // keep large host temporaries off the mmap/munmap (page-fault) path
  static bool done = false;
  if (!done) {
    mallopt(M_MMAP_THRESHOLD, 256 << 20);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
    done = true;
  }
}

void ensure_device() {
  tune_malloc();
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw Error(FMMLU_ECUDA, "no CUDA device available (libfmmlu has no CPU fallback)");
  }
}

// ---------------------------------------------------------------------------- cfg4: independent boxes
// BASELINE.json configs[3] (readings C21/C22): for each box, M = the 2n_γ proxy rows (Q = ∅),
// ID (id_stage), then the elimination of its redundant DOFs against its near set N, writing the
// box's Schur update Δ_{(S∪N)²} = −X_{(S∪N)R} X_RR⁻¹ X_{R(S∪N)} into a private buffer.  The same
// kernels as the tree path (k_proxy, Gram/pivoted Cholesky or TSQR/CPQR, k_trsm_T, k_build,
// DMMA GEMMs, Gauss-Jordan), processed in waves sized to free device memory.
double box_model_flops(int b, int kk, int nn, int m) {  // SURVEY §8(d) per-box cost model
  const double r = b - kk, K = kk, N = nn, B = b, Mr = m;
  const double kgen = 70.0 * (Mr * B + B * B + 2.0 * B * N);
  const double qr = 8.0 * Mr * B * B - (8.0 / 3.0) * B * B * B;
  const double cpqr = 8.0 * (B * B * K - B * K * K + K * K * K / 3.0) + 4.0 * K * K * r;
  const double ef = 8.0 * (3.0 * r * r * K + K * K * r) + 8.0 * r * K * K + 16.0 * r * K * N;
  const double pan = (8.0 / 3.0) * r * r * r + 16.0 * r * r * (K + N);
  const double schur = 8.0 * (K + N) * (K + N) * r;
  return kgen + qr + cpqr + (r > 0 ? ef + pan + schur : 0.0);
}

void boxes_impl(fmmlu_handle* h, const double* pts, const double* nrm, const double* npts, const double* nnrm,
                int nbox, int b, int nnear, double w, double k, double eps, int ngamma, double rho, int* ranks,
                int* perm, int nkeep, const int* keep_ids, void* delta, double* timing) {
  cudaStream_t st = h->stream;
  const int npb = b + nnear, m = 2 * ngamma;
  const double sg = std::sqrt(4.0 * M_PI * rho * rho / ngamma);
  std::unordered_map<int, int> kslot;
  for (int j = 0; j < nkeep; ++j) kslot[keep_ids[j]] = j;
  const bool in_dev = is_device_ptr(pts);
  const bool rk_dev = is_device_ptr(ranks), pm_dev = perm && is_device_ptr(perm),
             dl_dev = delta && is_device_ptr(delta);
  const long long tcap = (long long)(b / 2 + 1) * (b - b / 2 + 1);
  // per-box device bytes (upper bounds: k ≤ b for the factor pieces and Δ)
  const double per_box = 16.0 * ((double)m * b + 2.0 * b * b + (double)b * npb + (double)nnear * b + tcap +
                                 (double)npb * npb + (double)b * b + 2.0 * b * npb) +
                         8.0 * 13.0 * npb + 64.0 * b;
  size_t fr = 0, tot = 0;
  FMMLU_CUDA(cudaMemGetInfo(&fr, &tot));
  fr += big_cache(h->dev).cached();  // cached blocks are reusable (or evicted on demand)
  const int wave = (int)std::max(1.0, std::min<double>({(double)nbox, 1024.0, 0.45 * fr / per_box}));
  cudaEvent_t e0, e1;
  FMMLU_CUDA(cudaEventCreate(&e0));
  FMMLU_CUDA(cudaEventCreate(&e1));
  FMMLU_CUDA(cudaEventRecord(e0, st));
  double model = 0.0;
  DBuf status;
  status.alloc(16, st);
  FMMLU_CUDA(cudaMemsetAsync(status.p, 0, 16, st));
  const cplx m1 = cmk(-1.0, 0.0), p1 = cmk(1.0, 0.0);
  static const bool trace = getenv("FMMLU_TRACE") != nullptr;
  for (int w0 = 0; w0 < nbox; w0 += wave) {
    const double tw0 = now_ms(), ww0 = h->stats.t_sync_wait_ms;
    const int nw = std::min(wave, nbox - w0);
    const long long np = (long long)nw * npb;
    std::vector<DBuf> keep;
    // ---- geometry (SoA) of the wave
    DBuf gin, geo;
    const double *dp = pts + (size_t)w0 * b * 3, *dn = nrm + (size_t)w0 * b * 3,
                 *dq = npts + (size_t)w0 * nnear * 3, *dr = nnrm + (size_t)w0 * nnear * 3;
    if (!in_dev) {
      const size_t sb = (size_t)nw * b * 3 * sizeof(double), sn = (size_t)nw * nnear * 3 * sizeof(double);
      gin.alloc(2 * sb + 2 * sn, st);
      char* base = gin.as<char>();
      h2d(base, dp, sb, st);
      h2d(base + sb, dn, sb, st);
      h2d(base + 2 * sb, dq, sn, st);
      h2d(base + 2 * sb + sn, dr, sn, st);
      dp = (const double*)base;
      dn = (const double*)(base + sb);
      dq = (const double*)(base + 2 * sb);
      dr = (const double*)(base + 2 * sb + sn);
    }
    geo.alloc((size_t)7 * np * sizeof(double), st);
    double* G7 = geo.as<double>();
    launch_box_geo(dp, dn, dq, dr, nw, b, nnear, std::sqrt(w), G7, st);
    const Geo g{G7, G7 + np, G7 + 2 * np, G7 + 3 * np, G7 + 4 * np, G7 + 5 * np, G7 + 6 * np};
    // ---- M (proxy rows) and the ID
    DBuf M, Tb, permd, kd;
    IdAux aux;
    std::vector<cplx*> mp_keep;
    std::vector<int> pofs_keep;
    std::vector<long long> tofs_keep;
    M.alloc((size_t)nw * m * b * sizeof(cplx), st);
    Tb.alloc((size_t)nw * tcap * sizeof(cplx), st);
    permd.alloc((size_t)nw * b * sizeof(int), st);
    kd.alloc((size_t)nw * sizeof(int), st);
    {
      std::vector<int> gidx((size_t)nw * b);
      std::vector<ProxyTask> pt(nw);
      for (int j = 0; j < nw; ++j) {
        for (int t = 0; t < b; ++t) gidx[(size_t)j * b + t] = j * npb + t;
        ProxyTask q{};
        q.dst = (long long)j * m * b;
        q.ld = m;
        q.row0 = 0;
        q.b = b;
        q.idx_off = j * b;
        q.ngamma = ngamma;
        q.cx = q.cy = q.cz = 0.0;
        q.rho = rho;
        q.sg = sg;
        pt[j] = q;
      }
      Stage sg_;
      size_t o_p = sg_.add(pt), o_g = sg_.add(gidx);
      sg_.upload(st);
      int pid = h->prof.begin(FMMLU_K_GATHER, st);
      launch_proxy(sg_.ptr<ProxyTask>(o_p), nw, sg_.ptr<int>(o_g), M.as<cplx>(), g, k, st, ngamma);
      h->prof.end(pid, st);
      h->prof.add(FMMLU_K_GATHER, 120.0 * m * b * nw, 16.0 * m * b * nw, 1);
      keep.push_back(std::move(sg_.dev));
      std::vector<cplx*> mp(nw);
      std::vector<int> mrows(nw, m), bcol(nw, b), pofs(nw), mfin(nw);
      std::vector<long long> tofs(nw);
      for (int j = 0; j < nw; ++j) {
        mp[j] = M.as<cplx>() + (size_t)j * m * b;
        pofs[j] = j * b;
        tofs[j] = (long long)j * tcap;
      }
      id_stage(h, mp, mrows, bcol, pofs, tofs, eps, permd.as<int>(), kd.as<int>(), Tb.as<cplx>(), keep, mfin, &aux);
      mp_keep = mp;
      pofs_keep = pofs;
      tofs_keep = tofs;
    }
    std::vector<int> hk(nw), hp((size_t)nw * b);
    int* pin = h->d2h(nw + (size_t)nw * b);
    FMMLU_CUDA(cudaMemcpyAsync(pin, kd.p, nw * sizeof(int), cudaMemcpyDeviceToHost, st));
    FMMLU_CUDA(cudaMemcpyAsync(pin + nw, permd.p, (size_t)nw * b * sizeof(int), cudaMemcpyDeviceToHost, st));
    wait_stream(h, st);
    std::memcpy(hk.data(), pin, nw * sizeof(int));
    std::memcpy(hp.data(), pin + nw, (size_t)nw * b * sizeof(int));
    if (const char* dump = getenv("FMMLU_DEBUG_DUMP_T")) {  // diagnostics: T of the wave's first box
      std::vector<cplx> t0((size_t)hk[0] * (b - hk[0]));
      FMMLU_CUDA(cudaMemcpy(t0.data(), Tb.p, t0.size() * sizeof(cplx), cudaMemcpyDeviceToHost));
      if (FILE* f = fopen(dump, "wb")) {
        fwrite(t0.data(), sizeof(cplx), t0.size(), f);
        fclose(f);
      }
    }
    h->prof.resolve();
    // corrected-seminormal-equations steps: each contracts the T error by ≈ u·cond(M_S)² (R4)
    for (int it = 0; aux.gram && it < h->id_refine; ++it)
      refine_T(h, mp_keep, std::vector<int>(nw, m), std::vector<int>(nw, b), hk, hp, pofs_keep, Tb.as<cplx>(),
               tofs_keep, aux, keep);
    // ---- elimination
    std::vector<int> el;
    long long wsW = 0, wsF = 0, wsD = 0;
    std::vector<long long> oWB(nw), oWN(nw), oT(nw), oXi(nw), oUp(nw), oLp(nw), oD(nw);
    for (int j = 0; j < nw; ++j) {
      const int kk = hk[j], r = b - kk, kn = kk + nnear;
      model += box_model_flops(b, kk, nnear, m);
      if (r <= 0) continue;
      el.push_back(j);
      oWB[j] = wsW;
      wsW += (long long)b * npb;
      oWN[j] = wsW;
      wsW += (long long)nnear * b;
      oT[j] = wsF;
      wsF += (long long)kk * r;
      oXi[j] = wsF;
      wsF += (long long)r * r;
      oUp[j] = wsF;
      wsF += (long long)r * kn;
      oLp[j] = wsF;
      wsF += (long long)kn * r;
      oD[j] = wsD;
      wsD += (long long)kn * kn;
    }
    DBuf Wb, Fb, Db;
    Wb.alloc((size_t)std::max<long long>(wsW, 1) * sizeof(cplx), st);
    Fb.alloc((size_t)std::max<long long>(wsF, 1) * sizeof(cplx), st);
    Db.alloc((size_t)std::max<long long>(wsD, 1) * sizeof(cplx), st);
    // the GEMM store epilogue accumulates (C += αAB): Up/Lp and Δ start from zero
    FMMLU_CUDA(cudaMemsetAsync(Fb.p, 0, (size_t)std::max<long long>(wsF, 1) * sizeof(cplx), st));
    FMMLU_CUDA(cudaMemsetAsync(Db.p, 0, (size_t)std::max<long long>(wsD, 1) * sizeof(cplx), st));
    cplx *W = Wb.as<cplx>(), *Fp = Fb.as<cplx>(), *D = Db.as<cplx>();
    if (!el.empty()) {
      // W_B = Ã[B_RS, B_RS ∪ N] and W_N = Ã[N, B_RS] generated directly in [R | S] order
      std::vector<int> gl, slot, pos;
      std::vector<BuildTask> bt;
      std::vector<CopyTask> cpT, cpX;
      auto tiles = [&](long long dst, int ldd, int ro, int co, int ni, int nj) {
        for (int i0 = 0; i0 < ni; i0 += kTile)
          for (int j0 = 0; j0 < nj; j0 += kTile) {
            BuildTask t{};
            t.dst = dst;
            t.ldd = ldd;
            t.rows_off = ro;
            t.cols_off = co;
            t.i0 = i0;
            t.j0 = j0;
            t.ni = std::min(kTile, ni - i0);
            t.nj = std::min(kTile, nj - j0);
            t.ns = 1;
            bt.push_back(t);
          }
      };
      for (int j : el) {
        const int kk = hk[j], r = b - kk;
        const int* pm = &hp[(size_t)j * b];
        const int ro = (int)gl.size();  // [R | S] then N
        for (int i = kk; i < b; ++i) gl.push_back(j * npb + pm[i]);
        for (int i = 0; i < kk; ++i) gl.push_back(j * npb + pm[i]);
        for (int t = 0; t < nnear; ++t) gl.push_back(j * npb + b + t);
        tiles(oWB[j], b, ro, ro, b, npb);            // W_B: rows B_RS, cols [B_RS | N]
        tiles(oWN[j], nnear, ro + b, ro, nnear, b);  // W_N: rows N, cols B_RS
        CopyTask c{};
        c.src = (long long)j * tcap;
        c.lds = std::max(kk, 1);
        c.dst = oT[j];
        c.ldd = std::max(kk, 1);
        c.rows = kk;
        c.cols = r;
        c.rmap_off = c.cmap_off = -1;
        if (kk > 0) cpT.push_back(c);
        CopyTask x{};
        x.src = oWB[j];
        x.lds = b;
        x.dst = oXi[j];
        x.ldd = r;
        x.rows = r;
        x.cols = r;
        x.rmap_off = x.cmap_off = -1;
        cpX.push_back(x);
      }
      slot.assign(gl.size(), -1);
      pos.assign(gl.size(), 0);
      std::vector<long long> tab(1, -1);
      std::vector<int> bld(1, 0), maps(1, 0);
      split_copy_tasks(cpT);
      split_copy_tasks(cpX);
      Stage sb;
      size_t o_t = sb.add(bt), o_g = sb.add(gl), o_s = sb.add(slot), o_p = sb.add(pos), o_tb = sb.add(tab),
             o_bl = sb.add(bld), o_ct = sb.add(cpT), o_cx = sb.add(cpX), o_m = sb.add(maps);
      sb.upload(st);
      int bid = h->prof.begin(FMMLU_K_BUILD, st);
      launch_build(sb.ptr<BuildTask>(o_t), (int)bt.size(), sb.ptr<int>(o_g), sb.ptr<int>(o_s), sb.ptr<int>(o_p),
                   sb.ptr<long long>(o_tb), sb.ptr<int>(o_bl), nullptr, W, g, k, st);
      h->prof.end(bid, st);
      h->prof.add(FMMLU_K_BUILD, 70.0 * (double)wsW, 16.0 * (double)wsW, 1);
      launch_copy(sb.ptr<CopyTask>(o_ct), (int)cpT.size(), sb.ptr<int>(o_m), Tb.as<cplx>(), Fp, st);
      std::vector<GemmProblem> gp;
      std::vector<GemmGroup> gt;
      for (int j : el) {  // E: W_B[R,:] −= Tᵀ W_B[S,:]
        const int kk = hk[j], r = b - kk;
        GemmProblem P{};
        P.m = r;
        P.n = npb;
        P.k = kk;
        P.opA = kOpT;
        P.opB = kOpN;
        P.A = Fp + oT[j];
        P.lda = std::max(kk, 1);
        P.B = W + oWB[j] + r;
        P.ldb = b;
        P.C = W + oWB[j];
        P.ldc = b;
        add_gemm(gp, gt, P);
      }
      run_gemms(gp, gt, m1, 0, nullptr, st, keep, h->prof, FMMLU_K_EF);
      for (int j : el) {  // F: W_B[:,R] −= W_B[:,S] T ;  W_N[:,R] −= W_N[:,S] T
        const int kk = hk[j], r = b - kk;
        GemmProblem P{};
        P.m = b;
        P.n = r;
        P.k = kk;
        P.opA = kOpN;
        P.opB = kOpN;
        P.A = W + oWB[j] + (long long)r * b;
        P.lda = b;
        P.B = Fp + oT[j];
        P.ldb = std::max(kk, 1);
        P.C = W + oWB[j];
        P.ldc = b;
        add_gemm(gp, gt, P);
        GemmProblem Q = P;
        Q.m = nnear;
        Q.A = W + oWN[j] + (long long)r * nnear;
        Q.lda = nnear;
        Q.C = W + oWN[j];
        Q.ldc = nnear;
        add_gemm(gp, gt, Q);
      }
      run_gemms(gp, gt, m1, 0, nullptr, st, keep, h->prof, FMMLU_K_EF);
      launch_copy(sb.ptr<CopyTask>(o_cx), (int)cpX.size(), sb.ptr<int>(o_m), W, Fp, st);
      {
        std::vector<std::pair<cplx*, int>> mats;
        for (int j : el) mats.push_back({Fp + oXi[j], b - hk[j]});
        gj_blocked(h, mats, status.as<int>(), keep, FMMLU_K_INV);
      }
      for (int j : el) {  // Up = X_RR⁻¹ X_{R(S∪N)} ;  Lp = X_{(S∪N)R} X_RR⁻¹
        const int kk = hk[j], r = b - kk, kn = kk + nnear;
        GemmProblem P{};
        P.m = r;
        P.n = kn;
        P.k = r;
        P.opA = kOpN;
        P.opB = kOpN;
        P.A = Fp + oXi[j];
        P.lda = r;
        P.B = W + oWB[j] + (long long)r * b;
        P.ldb = b;
        P.C = Fp + oUp[j];
        P.ldc = r;
        add_gemm(gp, gt, P);
        if (kk > 0) {
          GemmProblem Q{};
          Q.m = kk;
          Q.n = r;
          Q.k = r;
          Q.opA = kOpN;
          Q.opB = kOpN;
          Q.A = W + oWB[j] + r;
          Q.lda = b;
          Q.B = Fp + oXi[j];
          Q.ldb = r;
          Q.C = Fp + oLp[j];
          Q.ldc = kn;
          add_gemm(gp, gt, Q);
        }
        GemmProblem R{};
        R.m = nnear;
        R.n = r;
        R.k = r;
        R.opA = kOpN;
        R.opB = kOpN;
        R.A = W + oWN[j];
        R.lda = nnear;
        R.B = Fp + oXi[j];
        R.ldb = r;
        R.C = Fp + oLp[j] + kk;
        R.ldc = kn;
        add_gemm(gp, gt, R);
      }
      run_gemms(gp, gt, p1, 0, nullptr, st, keep, h->prof, FMMLU_K_PANEL);
      for (int j : el) {  // Δ = −Lp · X_{R(S∪N)}  (private per-box buffer, C21)
        const int kk = hk[j], r = b - kk, kn = kk + nnear;
        GemmProblem P{};
        P.m = kn;
        P.n = kn;
        P.k = r;
        P.opA = kOpN;
        P.opB = kOpN;
        P.A = Fp + oLp[j];
        P.lda = kn;
        P.B = W + oWB[j] + (long long)r * b;
        P.ldb = b;
        P.C = D + oD[j];
        P.ldc = kn;
        add_gemm(gp, gt, P);
      }
      run_gemms(gp, gt, m1, 0, nullptr, st, keep, h->prof, FMMLU_K_SCHUR);
      keep.push_back(std::move(sb.dev));
      if (const char* dump = getenv("FMMLU_DEBUG_DUMP_W")) {  // diagnostics: W_B | W_N | Xi of el[0]
        const int j = el[0], r = b - hk[j];
        std::vector<cplx> t0((size_t)b * npb + (size_t)nnear * b + (size_t)r * r);
        FMMLU_CUDA(cudaStreamSynchronize(st));
        FMMLU_CUDA(cudaMemcpy(t0.data(), W + oWB[j], ((size_t)b * npb + (size_t)nnear * b) * sizeof(cplx),
                              cudaMemcpyDeviceToHost));
        FMMLU_CUDA(cudaMemcpy(t0.data() + (size_t)b * npb + (size_t)nnear * b, Fp + oXi[j], (size_t)r * r * sizeof(cplx),
                              cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(dump, "wb")) {
          fwrite(t0.data(), sizeof(cplx), t0.size(), f);
          fclose(f);
        }
      }
    }
    // ---- outputs of the wave
    if (rk_dev) h2d(ranks + w0, hk.data(), nw * sizeof(int), st);
    else std::memcpy(ranks + w0, hk.data(), nw * sizeof(int));
    if (perm) {
      if (pm_dev) FMMLU_CUDA(cudaMemcpyAsync(perm + (size_t)w0 * b, permd.p, (size_t)nw * b * sizeof(int),
                                             cudaMemcpyDeviceToDevice, st));
      else std::memcpy(perm + (size_t)w0 * b, hp.data(), (size_t)nw * b * sizeof(int));
    }
    if (delta)
      for (int j = 0; j < nw; ++j) {
        auto it = kslot.find(w0 + j);
        if (it == kslot.end()) continue;
        const int kk = hk[j], kn = kk + nnear;
        cplx* out = reinterpret_cast<cplx*>(delta) + (size_t)it->second * npb * npb;
        if (b - kk <= 0) {  // nothing eliminated: Δ = 0
          if (dl_dev) FMMLU_CUDA(cudaMemsetAsync(out, 0, (size_t)kn * kn * sizeof(cplx), st));
          else std::memset(out, 0, (size_t)kn * kn * sizeof(cplx));
          continue;
        }
        FMMLU_CUDA(cudaMemcpyAsync(out, D + oD[j], (size_t)kn * kn * sizeof(cplx),
                                   dl_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
      }
    wait_stream(h, st);
    h->prof.resolve();
    if (trace) {
      fprintf(stderr, "[fmmlu boxes] wave %d (%d boxes): %.1f ms (host %.1f, wait %.1f) | allocator: %.1f ms in %lld "
                      "calls (max %.1f), cached %.1f GB\n",
              w0 / wave, nw, now_ms() - tw0, now_ms() - tw0 - (h->stats.t_sync_wait_ms - ww0),
              h->stats.t_sync_wait_ms - ww0, g_ac.alloc_ms, g_ac.nalloc, g_ac.alloc_max, big_cache(h->dev).cached() / 1e9);
      g_ac = AllocClock{};
    }
  }
  if (trace) {
    fprintf(stderr, "[fmmlu boxes] gpu ms by class:");
    static const char* nm[10] = {"build", "gather", "qr", "cpqr", "ef", "inv", "panel", "schur", "root", "solve"};
    for (int c = 0; c < 10; ++c)
      if (h->prof.ms[c] > 0.005) fprintf(stderr, " %s %.1f", nm[c], h->prof.ms[c]);
    fprintf(stderr, "\n");
  }
  FMMLU_CUDA(cudaEventRecord(e1, st));
  int sing = 0;
  FMMLU_CUDA(cudaMemcpyAsync(&sing, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMMLU_CUDA(cudaStreamSynchronize(st));
  float t = 0.f;
  FMMLU_CUDA(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (timing) {
    timing[0] = t;
    timing[1] = model * 1e-9;
    timing[2] = wave;
  }
  if (sing) throw Error(FMMLU_ESINGULAR, "exactly singular X_RR pivot in fmmlu_boxes");
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int fmmlu_tree(const double* points, const double* normals, const double* weights, int64_t n,
               int leaf_max, fmmlu_handle** out) {
  if (out) *out = nullptr;
  if (!out || !points || !normals || !weights) return fail(FMMLU_EINVAL, "NULL argument");
  if (n < 1) return fail(FMMLU_EINVAL, "n must be >= 1");
  if (n > (int64_t)INT32_MAX / 4) return fail(FMMLU_EINVAL, "n too large");
  if (leaf_max < 1) return fail(FMMLU_EINVAL, "leaf_max must be >= 1");
  fmmlu_handle* h = nullptr;
  int rc = guarded([&] {
    ensure_device();
    double t0 = now_ms();
    static const bool trace = getenv("FMMLU_TRACE") != nullptr || getenv("FMMLU_TREE_TRACE") != nullptr;
    double tl[8] = {0}, tm = t0;
    auto lap = [&](int i) {  // FMMLU_TRACE: where the host time of fmmlu_tree goes
      const double t = now_ms();
      tl[i] += t - tm;
      tm = t;
    };
    h = new fmmlu_handle();
    FMMLU_CUDA(cudaGetDevice(&h->dev));
    FMMLU_CUDA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    order_after_legacy(h->stream);  // device inputs written on the legacy default stream are complete
    lap(0);
    h->n = n;
    cudaStream_t st = h->stream;
    // ---- device front end (reading C14/R1): the inputs stay on the device;
    // checks, bounding box, quantisation, Morton keys, the key sort and the tree-order geometry run
    // there, and only (perm, sorted q) come back for the box-level bookkeeping on the host
    DBuf dP, dN, dW;
    const double* P = points;
    const double* N = normals;
    const double* W = weights;
    auto upload = [&](const double* src, size_t cnt, DBuf& b) -> const double* {
      if (is_device_ptr(src)) return src;
      b.alloc(cnt * sizeof(double), st);
      FMMLU_CUDA(cudaMemcpyAsync(b.p, src, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
      return b.as<double>();
    };
    P = upload(points, 3 * (size_t)n, dP);
    N = upload(normals, 3 * (size_t)n, dN);
    W = upload(weights, (size_t)n, dW);
    const int nb = tree_scan_blocks(n);
    DBuf part;
    part.alloc((size_t)6 * nb * sizeof(double) + sizeof(int) * 4, st);
    int* dflag = reinterpret_cast<int*>(part.as<double>() + 6 * nb);
    FMMLU_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    launch_tree_scan(P, N, W, n, part.as<double>(), dflag, st);
    std::vector<double> hp(6 * (size_t)nb + 2);
    FMMLU_CUDA(cudaMemcpyAsync(hp.data(), part.p, (size_t)6 * nb * sizeof(double) + sizeof(int), cudaMemcpyDeviceToHost,
                               st));
    FMMLU_CUDA(cudaStreamSynchronize(st));
    lap(1);
    int hflag = 0;
    std::memcpy(&hflag, hp.data() + 6 * nb, sizeof(int));
    if (hflag & 1) throw Error(FMMLU_EINVAL, "weights must be finite and > 0");
    if (hflag & 2) throw Error(FMMLU_EINVAL, "normals must be unit vectors");
    if (hflag & 4) throw Error(FMMLU_EINVAL, "points must be finite");
    double mn[3], mx[3], lo[3], side;
    for (int a = 0; a < 3; ++a) {
      mn[a] = hp[a];
      mx[a] = hp[3 + a];
      for (int b = 1; b < nb; ++b) {
        mn[a] = std::min(mn[a], hp[6 * b + a]);
        mx[a] = std::max(mx[a], hp[6 * b + 3 + a]);
      }
    }
    Tree::root_cube(mn, mx, lo, side);
    DBuf keys, idx, qb;
    keys.alloc(2 * (size_t)n * sizeof(unsigned long long), st);
    idx.alloc(2 * (size_t)n * sizeof(int), st);
    qb.alloc(6 * (size_t)n * sizeof(int), st);  // q (input order) | q (tree order)
    unsigned long long* k_in = keys.as<unsigned long long>();
    unsigned long long* k_out = k_in + n;
    int* i_in = idx.as<int>();
    int* i_out = i_in + n;
    int* q_in = qb.as<int>();
    int* q_out = q_in + 3 * n;
    launch_tree_keys(P, n, lo, side, k_in, i_in, q_in, st);
    size_t tmpb = 0;
    FMMLU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmpb, k_in, k_out, i_in, i_out, (int)n, 0, 3 * kDepth, st));
    DBuf tmp;
    tmp.alloc(std::max<size_t>(tmpb, 16), st);
    // stable LSD radix sort of (key, index): ties stay in index order, as the host's stable order
    FMMLU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmpb, k_in, k_out, i_in, i_out, (int)n, 0, 3 * kDepth, st));
    h->geo.alloc(7 * (size_t)n * sizeof(double), st);
    h->perm.alloc(n * sizeof(long long), st);
    launch_tree_gather(P, N, W, n, i_out, q_in, h->geo.as<double>(), h->perm.as<long long>(), q_out, st);
    lap(2);
    // boxes: subdivision + 2:1 balance on the device from the sorted keys (devtree.cu); the host
    // receives the per-level box arrays for the owner / list bookkeeping
    DevTreeResult dt;
    int dt_launches = 0;
    device_octree(k_out, n, leaf_max, st, dt, &dt_launches);
    lap(3);
    int* hperm = h->d2h(n);  // pinned landing buffer (a pageable copy is staged by the driver)
    FMMLU_CUDA(cudaMemcpyAsync(hperm, i_out, n * sizeof(int), cudaMemcpyDeviceToHost, st));
    FMMLU_CUDA(cudaStreamSynchronize(st));
    lap(4);
    h->tree.build_from_levels(dt.level_n, dt.code, dt.start, dt.end, dt.parent, hperm, lo, side, n, leaf_max);
    {
      // device copy of the finished tree for the owner-list kernels (build_topo)
      const int nbx = (int)h->tree.boxes.size();
      std::vector<unsigned char> leaf(nbx);
      for (int b = 0; b < nbx; ++b) leaf[b] = h->tree.boxes[b].leaf() ? 1 : 0;
      h->level_first.assign(h->tree.nlevels + 1, 0);
      for (int l = 0; l < h->tree.nlevels; ++l) h->level_first[l + 1] = h->level_first[l] + dt.level_n[l];
      h->tcode.alloc((size_t)nbx * sizeof(unsigned long long), st);
      h->tleaf.alloc((size_t)nbx, st);
      h->tleafrank.alloc((size_t)(nbx + 1) * sizeof(int), st);
      FMMLU_CUDA(cudaMemcpyAsync(h->tcode.p, dt.code.data(), (size_t)nbx * sizeof(unsigned long long),
                                 cudaMemcpyHostToDevice, st));
      FMMLU_CUDA(cudaMemcpyAsync(h->tleaf.p, leaf.data(), (size_t)nbx, cudaMemcpyHostToDevice, st));
      device_leafrank(h->tleaf.as<unsigned char>(), nbx, h->tleafrank.as<int>(), st);
      FMMLU_CUDA(cudaStreamSynchronize(st));
    }
    lap(5);
    // k_tree_scan/keys/gather + CUB onesweep radix sort (histogram + 8 passes) + device octree
    h->tree_launches = 3 + 9 + dt_launches;
    double* gp = h->geo.as<double>();
    h->g = Geo{gp, gp + n, gp + 2 * n, gp + 3 * n, gp + 4 * n, gp + 5 * n, gp + 6 * n};
    track(h, h->geo.bytes + h->perm.bytes);
    fmmlu_stats_t& S = h->stats;
    S.n = n;
    S.nlevels = h->tree.nlevels;
    S.nboxes = (int)h->tree.boxes.size();
    S.nleaves = 0;
    for (auto& b : h->tree.boxes) S.nleaves += b.leaf();
    S.t_tree_ms = now_ms() - t0;
    if (trace) {
      fprintf(stderr, "[fmmlu] tree host ms: stream+order %.1f scan+sync %.1f keys/sort/gather launch %.1f octree %.1f "
                      "perm d2h %.1f boxes %.1f | total %.1f | allocator %.1f ms in %lld calls (max %.1f)\n",
              tl[0], tl[1], tl[2], tl[3], tl[4], tl[5], S.t_tree_ms, g_ac.alloc_ms, g_ac.nalloc, g_ac.alloc_max);
      g_ac = AllocClock{};
    }
  });
  if (rc != FMMLU_OK) {
    if (h) fmmlu_destroy(h);
    return rc;
  }
  *out = h;
  return FMMLU_OK;
}

int fmmlu_factor(fmmlu_handle* h, double k, double eps) {
  if (!h) return fail(FMMLU_EINVAL, "NULL handle");
  if (!(k > 0.0) || !std::isfinite(k)) return fail(FMMLU_EINVAL, "k must be finite and > 0");
  if (!(eps > 0.0 && eps < 1.0)) return fail(FMMLU_EINVAL, "eps must lie in (0, 1)");
  return guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    double t0 = now_ms();
    tl_pin.reset();
    h->prof.reset();
    h->stats.t_sync_wait_ms = 0;
    factor_impl(h, k, eps);
    h->stats.t_factor_ms = now_ms() - t0;
    h->stats.peak_bytes = (int64_t)h->peak_bytes;
  });
}

int fmmlu_solve(fmmlu_handle* h, void* rhs, int nrhs) {
  if (!h) return fail(FMMLU_EINVAL, "NULL handle");
  if (!rhs) return fail(FMMLU_EINVAL, "NULL rhs");
  if (nrhs < 1) return fail(FMMLU_EINVAL, "nrhs must be >= 1");
  if (!h->factored) return fail(FMMLU_ESTATE, "fmmlu_solve called before a successful fmmlu_factor");
  return guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    if (h->stream == h->own_stream) order_after_legacy(h->stream);
    double t0 = now_ms();
    solve_impl(h, rhs, nrhs);
    h->stats.t_solve_ms = now_ms() - t0;
  });
}

int fmmlu_apply(fmmlu_handle* h, void* x, int nrhs) {
  if (!h) return fail(FMMLU_EINVAL, "NULL handle");
  if (!x) return fail(FMMLU_EINVAL, "NULL x");
  if (nrhs < 1) return fail(FMMLU_EINVAL, "nrhs must be >= 1");
  if (!h->factored) return fail(FMMLU_ESTATE, "fmmlu_apply called before a successful fmmlu_factor");
  return guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    if (h->stream == h->own_stream) order_after_legacy(h->stream);
    apply_impl(h, x, nrhs);
  });
}

// Monostatic sonar cross section (§6.3, reading R8): for each azimuth φ_a the
// plane-wave system A σ = −e^{ik x·d_a} is solved with the stored factors and
// R(φ_a) = (−ik/4π) Σ_j w_j (1 − n_j·d_a) e^{ik x_j·d_a} σ_j.  Everything stays in tree order on the
// device: the RHS is generated already W^{½}-scaled and R is reduced from y = W^{½}σ directly.
void rcs_impl(fmmlu_handle* h, const double* phis, int nphi, void* Rout) {
  cudaStream_t st = h->stream;
  const int n = (int)h->n;
  DBuf dphi, dR;
  const double* ph = phis;
  if (!is_device_ptr(phis)) {
    dphi.alloc((size_t)nphi * sizeof(double), st);
    FMMLU_CUDA(cudaMemcpyAsync(dphi.p, phis, (size_t)nphi * sizeof(double), cudaMemcpyHostToDevice, st));
    ph = dphi.as<double>();
  }
  const bool rdev = is_device_ptr(Rout);
  cplx* R = reinterpret_cast<cplx*>(Rout);
  if (!rdev) {
    dR.alloc((size_t)nphi * sizeof(cplx), st);
    R = dR.as<cplx>();
  }
  FMMLU_CUDA(cudaMemsetAsync(R, 0, (size_t)nphi * sizeof(cplx), st));
  const bool gemm_sweeps = use_gemm_sweeps(h, nphi);
  const int qc = gemm_sweeps ? sweep_chunk(h, nphi) : nphi;
  DBuf yb;
  yb.alloc((size_t)n * qc * sizeof(cplx), st);
  cplx* y = yb.as<cplx>();
  for (int a0 = 0; a0 < nphi; a0 += qc) {
    const int q = std::min(qc, nphi - a0);
    int id = h->prof.begin(FMMLU_K_SOLVE, st);
    launch_plane_wave(h->g, n, h->k, ph + a0, q, y, n, st);
    h->prof.end(id, st);
    if (gemm_sweeps) {
      sweeps_gemm(h, y, n, q);
    } else {  // few angles: the per-box solve kernels (the same path as fmmlu_solve)
      size_t scr_rows = 1;
      for (auto& p : h->phases) scr_rows = std::max(scr_rows, (size_t)p.tmp_rows);
      DBuf scr, tmp;
      scr.alloc(scr_rows * q * sizeof(cplx), st);
      id = h->prof.begin(FMMLU_K_SOLVE, st);
      sweeps_boxes(h, y, n, q, scr.as<cplx>(), st);
      h->prof.end(id, st);
      wait_stream(h, st);
    }
    id = h->prof.begin(FMMLU_K_SOLVE, st);
    launch_rcs_reduce(h->g, n, h->k, ph + a0, q, y, n, R + a0, st);
    h->prof.end(id, st);
  }
  if (!rdev) FMMLU_CUDA(cudaMemcpyAsync(Rout, R, (size_t)nphi * sizeof(cplx), cudaMemcpyDeviceToHost, st));
  wait_stream(h, st);
  h->prof.resolve();
}

int fmmlu_monostatic_rcs(fmmlu_handle* h, const double* phis, int nphi, void* R) {
  if (!h) return fail(FMMLU_EINVAL, "NULL handle");
  if (!phis || !R) return fail(FMMLU_EINVAL, "NULL phis / R");
  if (nphi < 1) return fail(FMMLU_EINVAL, "nphi must be >= 1");
  if (!h->factored) return fail(FMMLU_ESTATE, "fmmlu_monostatic_rcs called before a successful fmmlu_factor");
  return guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    if (h->stream == h->own_stream) order_after_legacy(h->stream);
    double t0 = now_ms();
    rcs_impl(h, phis, nphi, R);
    h->stats.t_solve_ms = now_ms() - t0;
  });
}

int fmmlu_matvec(fmmlu_handle* h, double k, const void* x, void* y, int nrhs) {
  if (!h) return fail(FMMLU_EINVAL, "NULL handle");
  if (!x || !y || nrhs < 1) return fail(FMMLU_EINVAL, "bad x/y/nrhs");
  if (!std::isfinite(k) || k < 0) return fail(FMMLU_EINVAL, "k must be finite and >= 0");
  return guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    if (h->stream == h->own_stream) order_after_legacy(h->stream);
    cudaStream_t st = h->stream;
    const int n = (int)h->n;
    size_t bytes = (size_t)n * nrhs * sizeof(cplx);
    DBuf xi, xt, yt;
    const cplx* xs = reinterpret_cast<const cplx*>(x);
    if (!is_device_ptr(x)) {
      xi.alloc(bytes, st);
      FMMLU_CUDA(cudaMemcpyAsync(xi.p, x, bytes, cudaMemcpyHostToDevice, st));
      xs = xi.as<cplx>();
    }
    xt.alloc(bytes, st);
    yt.alloc(bytes, st);
    launch_permute_in(xs, n, xt.as<cplx>(), n, nrhs, h->perm.as<long long>(), h->g.sw, 0, st);
    launch_matvec(h->g, k, n, xt.as<cplx>(), yt.as<cplx>(), nrhs, st);
    if (is_device_ptr(y)) {
      launch_permute_out(yt.as<cplx>(), reinterpret_cast<cplx*>(y), n, n, nrhs, h->perm.as<long long>(), h->g.sw, 0,
                         st);
    } else {
      launch_permute_out(yt.as<cplx>(), xt.as<cplx>(), n, n, nrhs, h->perm.as<long long>(), h->g.sw, 0, st);
      FMMLU_CUDA(cudaMemcpyAsync(y, xt.p, bytes, cudaMemcpyDeviceToHost, st));
    }
    FMMLU_CUDA(cudaStreamSynchronize(st));
  });
}

int fmmlu_inverse_batch(fmmlu_handle* h, void* A, int n, int count, double* ms) {
  if (!h || !A) return fail(FMMLU_EINVAL, "NULL argument");
  if (n < 1 || count < 1) return fail(FMMLU_EINVAL, "n and count must be >= 1");
  if (!is_device_ptr(A)) return fail(FMMLU_EINVAL, "A must be a device pointer");
  int sing = 0;
  int rc = guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    cudaStream_t st = h->stream;
    DBuf status;
    status.alloc(16, st);
    FMMLU_CUDA(cudaMemsetAsync(status.p, 0, 16, st));
    std::vector<std::pair<cplx*, int>> mats;
    for (int c = 0; c < count; ++c) mats.push_back({reinterpret_cast<cplx*>(A) + (size_t)c * n * n, n});
    std::vector<DBuf> keep;
    h->prof.resolve();
    const double before = h->prof.ms[FMMLU_K_INV];
    gj_blocked(h, mats, status.as<int>(), keep, FMMLU_K_INV);  // events bracket the kernels only
    FMMLU_CUDA(cudaMemcpyAsync(&sing, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FMMLU_CUDA(cudaStreamSynchronize(st));
    h->prof.resolve();
    if (ms) *ms = h->prof.ms[FMMLU_K_INV] - before;
  });
  if (rc != FMMLU_OK) return rc;
  if (sing) return fail(FMMLU_ESINGULAR, "exactly singular pivot in fmmlu_inverse_batch");
  return FMMLU_OK;
}

int fmmlu_boxes(const double* pts, const double* nrm, const double* npts, const double* nnrm, int nbox, int b,
                int nnear, double w, double k, double eps, int n_gamma, double rho, int* ranks, int* perm,
                int nkeep, const int* keep, void* delta, double* timing) {
  if (!pts || !nrm || !npts || !nnrm || !ranks) return fail(FMMLU_EINVAL, "NULL argument");
  if (nbox < 1 || b < 1 || nnear < 0 || n_gamma < 1) return fail(FMMLU_EINVAL, "bad sizes");
  if (!(w > 0) || !(rho > 0) || !std::isfinite(k) || k < 0) return fail(FMMLU_EINVAL, "bad w / rho / k");
  if (!(eps > 0 && eps < 1)) return fail(FMMLU_EINVAL, "eps must lie in (0, 1)");
  if (nkeep < 0 || (nkeep > 0 && (!keep || !delta))) return fail(FMMLU_EINVAL, "bad keep / delta");
  for (int j = 0; j < nkeep; ++j)
    if (keep[j] < 0 || keep[j] >= nbox) return fail(FMMLU_EINVAL, "keep id out of range");
  fmmlu_handle* h = nullptr;
  int rc = guarded([&] {
    ensure_device();
    h = new fmmlu_handle();
    FMMLU_CUDA(cudaGetDevice(&h->dev));
    FMMLU_CUDA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    order_after_legacy(h->stream);
    // Δ is this workload's output and multiplies T by A_SS: T must be accurate to ≈ u·cond(M_S).
    // Gram path (ε ≥ 1e-7) + one corrected-seminormal-equations step gives that at GEMM speed;
    // the Householder path (ε < 1e-7) has it by construction.
    h->id_mode = 0;
    h->id_refine = 2;
    h->pchol_ll = getenv("FMMLU_BOXES_LL") ? atoi(getenv("FMMLU_BOXES_LL")) : 0;  // cfg4 ranks are ≈ b
    if (const char* e = getenv("FMMLU_BOXES_ID_MODE")) h->id_mode = atoi(e);
    if (const char* e = getenv("FMMLU_BOXES_REFINE")) h->id_refine = atoi(e);
    boxes_impl(h, pts, nrm, npts, nnrm, nbox, b, nnear, w, k, eps, n_gamma, rho, ranks, perm, nkeep, keep, delta,
               timing);
  });
  if (h) {
    for (auto& w : h->ws_slot) w.release();  // stream-ordered frees need the stream alive
    cudaStreamSynchronize(h->stream);
    if (h->own_stream) {
      drop_arena(h->own_stream);
      cudaStreamDestroy(h->own_stream);
    }
    delete h;
  }
  return rc;
}

int fmmlu_destroy(fmmlu_handle* h) {
  if (!h) return FMMLU_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(h->dev);  // blocks go back to this device's cache / pool, events on its streams
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->phases.clear();
  h->fac_chunks.clear();
  h->root.release();
  h->root_rows.release();
  h->root_rows_in.release();
  h->root_dinv.release();
  h->root_flags.release();
  h->sep_perm.release();
  h->drop_solve_graphs();
  h->sv_y.release();
  h->sv_scr.release();
  h->sv_root.release();
  h->tcode.release();
  h->tleaf.release();
  h->tleafrank.release();
  for (auto& w : h->ws_slot) w.release();
  h->geo.release();
  h->perm.release();
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->own_stream) {
    drop_arena(h->own_stream);
    cudaStreamDestroy(h->own_stream);
  }
  delete h;
  if (prev >= 0) cudaSetDevice(prev);
  return FMMLU_OK;
}

int fmmlu_release_cache(void) {
  return guarded([&] {
    int ndev = 0, prev = 0;
    FMMLU_CUDA(cudaGetDeviceCount(&ndev));
    FMMLU_CUDA(cudaGetDevice(&prev));
    for (int d = 0; d < std::min(ndev, kMaxDev); ++d) {
      FMMLU_CUDA(cudaSetDevice(d));
      release_dev_work(d);
      big_cache(d).flush(nullptr);
      FMMLU_CUDA(cudaDeviceSynchronize());
      FMMLU_CUDA(cudaMemPoolTrimTo(lib_pool(d), 0));
    }
    FMMLU_CUDA(cudaSetDevice(prev));
  });
}

const char* fmmlu_last_error(void) { return g_last_error.c_str(); }

int fmmlu_stats(const fmmlu_handle* h, fmmlu_stats_t* out) {
  if (!h || !out) return fail(FMMLU_EINVAL, "NULL argument");
  *out = h->stats;
  out->peak_bytes = (int64_t)h->peak_bytes;
  out->n_launches = h->prof.total_launches + h->tree_launches + h->topo_launches.load();
  for (int i = 0; i < 16; ++i) {
    out->class_ms[i] = h->prof.ms[i];
    out->class_flops[i] = h->prof.flops[i];
    out->class_bytes[i] = h->prof.bytes[i];
    out->class_launches[i] = h->prof.launches[i];
  }
  return FMMLU_OK;
}

int fmmlu_set_stream(fmmlu_handle* h, void* s) {
  if (!h) return fail(FMMLU_EINVAL, "NULL handle");
  h->stream = s ? reinterpret_cast<cudaStream_t>(s) : h->own_stream;
  return FMMLU_OK;
}

int fmmlu_set_param(fmmlu_handle* h, const char* name, double value) {
  if (!h || !name) return fail(FMMLU_EINVAL, "NULL argument");
  std::string k(name);
  if (k == "id_mode") {
    if (value != 0 && value != 1 && value != 2 && value != 3)
      return fail(FMMLU_EINVAL, "id_mode must be 0, 1, 2 or 3");
    h->id_mode = (int)value;
  } else if (k == "pchol_mode") {
    if (value != 0 && value != 1) return fail(FMMLU_EINVAL, "pchol_mode must be 0 or 1");
    h->pchol_mode = (int)value;
  } else if (k == "id_refine") {
    if (!(value >= 0 && value <= 3 && value == (int)value)) return fail(FMMLU_EINVAL, "id_refine must be 0..3");
    h->id_refine = (int)value;
  } else if (k == "gj_mode") {
    if (value != 0 && value != 1) return fail(FMMLU_EINVAL, "gj_mode must be 0 or 1");
    h->gj_mode = (int)value;
  } else if (k == "separate_id") {
    if (value != 0 && value != 1) return fail(FMMLU_EINVAL, "separate_id must be 0 or 1");
    h->separate_id = (int)value;
  } else if (k == "deterministic") {
    if (value != 0 && value != 1) return fail(FMMLU_EINVAL, "deterministic must be 0 or 1");
    h->deterministic = (int)value;
  } else if (k == "proxy_rho") {
    if (!(value > 0.87 && value < 2.5)) return fail(FMMLU_EINVAL, "proxy_rho must lie in (0.87, 2.5)");
    h->rho_factor = value;
  } else {
    return fail(FMMLU_EINVAL, "unknown parameter " + k);
  }
  return FMMLU_OK;
}

int fmmlu_tree_boxes(const fmmlu_handle* h, int32_t* nboxes, int32_t* level, int32_t* coord, int32_t* start,
                     int32_t* end) {
  if (!h || !nboxes) return fail(FMMLU_EINVAL, "NULL argument");
  const int nb = (int)h->tree.boxes.size();
  if (!level && !coord && !start && !end) {
    *nboxes = nb;
    return FMMLU_OK;
  }
  if (*nboxes < nb) return fail(FMMLU_EINVAL, "box arrays too small");
  for (int b = 0; b < nb; ++b) {
    const Box& B = h->tree.boxes[b];
    if (level) level[b] = B.level;
    if (coord)
      for (int a = 0; a < 3; ++a) coord[3 * b + a] = B.c[a];
    if (start) start[b] = B.start;
    if (end) end[b] = B.end;
  }
  *nboxes = nb;
  return FMMLU_OK;
}

int fmmlu_level_lists(fmmlu_handle* h, int level, int32_t* counts, int32_t* owners, int32_t* nptr, int32_t* nidx,
                      int32_t* qptr, int32_t* qidx) {
  if (!h || !counts) return fail(FMMLU_EINVAL, "NULL argument");
  if (level < 2 || level >= h->tree.nlevels) return fail(FMMLU_EINVAL, "level out of range");
  return guarded([&] {
    FMMLU_CUDA(cudaSetDevice(h->dev));
    const int L = h->tree.nlevels;
    if ((int)h->topo.size() < L) h->topo.resize(L);
    if (h->topo_ready.size() < (size_t)L) h->topo_ready.resize(L, 0);
    if (!h->topo_ready[level]) {
      build_topo(h, level, h->topo[level]);
      h->topo_ready[level] = 1;
    }
    const LevelTopo& tp = h->topo[level];
    const int nlb = (int)tp.boxN.size(), no = (int)tp.owners.size();
    long long tn = 0, tq = 0;
    for (int i = 0; i < nlb; ++i) {
      tn += (long long)tp.boxN[i].size();
      tq += (long long)tp.boxQ[i].size();
    }
    counts[0] = nlb;
    counts[1] = no;
    counts[2] = (int32_t)tn;
    counts[3] = (int32_t)tq;
    if (!owners) return;
    if (!nptr || !nidx || !qptr || !qidx) throw Error(FMMLU_EINVAL, "NULL list array");
    std::copy(tp.owners.begin(), tp.owners.end(), owners);
    int a = 0, b = 0;
    for (int i = 0; i < nlb; ++i) {
      nptr[i] = a;
      qptr[i] = b;
      for (int o : tp.boxN[i]) nidx[a++] = o;
      for (int o : tp.boxQ[i]) qidx[b++] = o;
    }
    nptr[nlb] = a;
    qptr[nlb] = b;
  });
}

int fmmlu_tree_perm(const fmmlu_handle* h, int64_t* perm) {
  if (!h || !perm) return fail(FMMLU_EINVAL, "NULL argument");
  std::memcpy(perm, h->tree.perm.data(), h->n * sizeof(int64_t));
  return FMMLU_OK;
}

int fmmlu_probe_fp64(int kind, double* tflops) {
  if (!tflops || (kind != 0 && kind != 1)) return fail(FMMLU_EINVAL, "bad argument");
  return guarded([&] {
    ensure_device();
    *tflops = probe_fp64(kind);
  });
}

}  // extern "C"
