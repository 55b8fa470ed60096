// mrrr.cu -- host orchestrator and C ABI (include/mrrr.h) of the B200-native
// MRRR tridiagonal eigensolver.  The orchestrator plans launches (blocks,
// slots, tree levels, work chunks) from small read-backs; every arithmetic
// step of the method runs in the kernels of kernels_tree.cuh (root, bisection,
// classification), kernels_child.cuh (the cluster step) and kernels_warp.cuh
// (twisted factorizations and vectors).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <dlfcn.h>
#include <cstring>
#include <chrono>
#include <mutex>
#include <numeric>
#include <vector>

#include <cub/device/device_segmented_radix_sort.cuh>
#include <nvtx3/nvToolsExt.h>

#include "../../include/mrrr.h"
#include "kernels_tree.cuh"
#include "kernels_vec.cuh"
#include "kernels_warp.cuh"
#include "kernels_child.cuh"
#include "kernels_child2.cuh"
#include "kernels_child3.cuh"

using namespace mrrr;


namespace {

thread_local mrrr_stats_t g_stats;
thread_local int64_t g_rqc_hist[16];  // the calling thread's last solve (mrrr_get_rqc_histogram)

struct CudaError {
  cudaError_t e;
};
#define CK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) throw CudaError{e_}; \
  } while (0)
struct MrrrError {
  int code;
};

// Library-owned stream-ordered memory pool per device.  Its release threshold
// is unlimited, so workspace freed at the end of a call stays mapped for the
// next call instead of being returned to the driver at every synchronisation
// (the default pool's behaviour, which costs a remap of the whole workspace
// per call).  mrrr_trim_workspace() releases it.
cudaMemPool_t g_pools[64];
std::mutex g_pool_mu;

cudaMemPool_t lib_pool() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps pr{};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    CK(cudaMemPoolCreate(&g_pools[dev], &pr));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return g_pools[dev];
}

// Debug dump of device arrays (MRRR_DUMP=<dir>): raw little-endian files.
template <class T>
void dump(const char *name, const T *dptr, size_t count, cudaStream_t s) {
  const char *dir = getenv("MRRR_DUMP");
  if (!dir || !count) return;
  std::vector<T> h(count);
  CK(cudaMemcpyAsync(h.data(), dptr, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  char path[512];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE *f = fopen(path, "wb");
  if (f) { fwrite(h.data(), sizeof(T), count, f); fclose(f); }
}

// Per-thread library objects (streams, workspace, events, staging) are
// created on first use per device and RELEASED when the thread exits (the
// holders' destructors), so threads that call the library and exit leak
// nothing; mrrr_trim_workspace() releases the memory of the calling thread
// earlier.  (At process exit the CUDA context may already be gone; the
// destructors then ignore the errors.)
// Hardware work queues.  A CUDA context maps its streams onto
// CUDA_DEVICE_MAX_CONNECTIONS hardware queues (8 by default); a solve uses up
// to 11 streams of its own (below) next to the caller's, and two streams that
// share a queue wait for one another.  Measured on one B200 (random n = 20000,
// profiles/r02/setF): with 8 queues the tree stream's flag read-back after the
// last level's refinement returned only when an unrelated vector piece ended
// (~1 ms), and a piece launched on an idle side stream started only when an
// earlier piece on another stream ended; with 32 queues neither happens
// (34.2 -> 33.8 ms with four side streams, 32.5 ms with eight).  The variable
// is read when the context is created, so the library sets it (without
// overriding the caller's value) when it is loaded; a process that created its
// context earlier keeps its own setting and the solve is only slower.
__attribute__((constructor)) static void mrrr_on_load() { setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0); }

constexpr int kSide = 8;  // side streams for the vector batches (at most; MRRR_NSIDE of them are used)
constexpr int kNSideDefault = 8;  // with 32 hardware queues (above): 4 / 6 / 8 -> 33.7 / 32.8 / 32.6 ms at random n=20000, other configs unchanged
struct StreamSet {
  cudaStream_t st[64][kSide + 3] = {};  // per device: kSide side streams, the copy stream, the solve stream, the tree's second stream
  ~StreamSet() {
    for (auto &dv : st)
      for (cudaStream_t &x : dv)
        if (x) { cudaStreamDestroy(x); x = nullptr; }
  }
};
thread_local StreamSet g_streams;

cudaStream_t *side_streams() {
  int d = 0;
  CK(cudaGetDevice(&d));
  cudaStream_t *x = g_streams.st[d & 63];
  if (!x[0])
    for (int k = 0; k < kSide; ++k) CK(cudaStreamCreateWithFlags(&x[k], cudaStreamNonBlocking));
  return x;
}

cudaStream_t copy_stream() {  // Z downloads of the host entry (per thread and device)
  int d = 0;
  CK(cudaGetDevice(&d));
  cudaStream_t &x = g_streams.st[d & 63][kSide];
  if (!x) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  return x;
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Host wall-clock trace of the phases (MRRR_TRACE=1), for overhead hunting,
// and NVTX ranges of the same phases (always; header-only NVTX v3, a no-op
// unless a profiler injects itself): "mrrr" around the call, one nested
// range per phase (root, each tree level, the vector tail), one per vector
// piece launch.
struct NvtxScope {
  explicit NvtxScope(const char *name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
struct Trace {
  bool on;
  int lvl = 0;
  bool phase_open = false;
  std::chrono::steady_clock::time_point t0, tl;
  Trace() : on(getenv("MRRR_TRACE") != nullptr) {
    t0 = tl = std::chrono::steady_clock::now();
    if (on) lvl = atoi(getenv("MRRR_TRACE"));
    nvtxRangePushA("mrrr");
  }
  ~Trace() {
    if (phase_open) nvtxRangePop();
    nvtxRangePop();
  }
  void phase(const char *name) {
    if (phase_open) nvtxRangePop();
    nvtxRangePushA(name);
    phase_open = true;
  }
  // MRRR_TRACE=2: also the steps inside a tree level (synchronising the stream)
  void fine(cudaStream_t s, const char *what) {
    if (lvl < 2) return;
    cudaStreamSynchronize(s);
    mark(what);
  }
  void mark(const char *what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[mrrr] %-28s +%8.3f ms  (at %8.3f ms)\n", what,
            std::chrono::duration<double, std::milli>(t - tl).count(),
            std::chrono::duration<double, std::milli>(t - t0).count());
    tl = t;
  }
};

// Device workspace: per-thread, per-device bump allocators over chunks that
// are kept across calls.  A solve allocates from two of them: the CALL
// workspace (reset when a call starts; everything that lives until the
// vectors) and the LEVEL workspace (reset at every tree level; probe scratch,
// cluster lists, work items).  Reuse is safe by stream order: a call
// synchronises its stream (and joins its side stream) before returning, and
// level L+1's uploads and kernels follow level L's on the call's stream.  In
// steady state no call allocates device memory at all: the stream-ordered
// pool this replaces grew (remapped) at unpredictable levels, which cost up
// to a second inside a level (MRRR_TRACE=2, n = 1e5) and 100-700 ms outliers
// per solve at n = 20000.  mrrr_trim_workspace() frees the chunks.
struct BumpWs {
  std::vector<std::pair<char *, size_t>> chunks;
  size_t chunk = 0, off = 0;
  size_t used = 0, used_peak = 0;  // bytes handed out since the last reset, and their peak over resets
  void *get(size_t bytes) {
    bytes = (std::max<size_t>(bytes, 1) + 255) & ~size_t(255);
    used += bytes;
    used_peak = std::max(used_peak, used);
    for (;;) {
      if (chunk < chunks.size() && off + bytes <= chunks[chunk].second) {
        void *p = chunks[chunk].first + off;
        off += bytes;
        return p;
      }
      if (chunk + 1 < chunks.size()) { ++chunk; off = 0; continue; }
      // geometric growth up to 1 GiB chunks; a larger request gets its own size
      size_t sz = std::max<size_t>(bytes, chunks.empty() ? (size_t(64) << 20)
                                                         : std::min<size_t>(2 * chunks.back().second, size_t(1) << 30));
      char *p = nullptr;
      cudaError_t e = cudaMalloc((void **)&p, sz);
      if (e == cudaErrorMemoryAllocation && sz > bytes) {
        cudaGetLastError();
        sz = bytes;
        e = cudaMalloc((void **)&p, sz);
      }
      if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); throw MrrrError{MRRR_ERR_NOMEM}; }
      CK(e);
      chunks.push_back({p, sz});
      chunk = chunks.size() - 1;
      off = 0;
    }
  }
  void reset() { chunk = 0; off = 0; used = 0; }
  void release() {
    for (auto &c : chunks) cudaFree(c.first);
    chunks.clear();
    reset();
  }
  ~BumpWs() { release(); }
};
thread_local BumpWs g_ws_call[64], g_ws_level[64];

BumpWs &device_ws(BumpWs *arr) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  return arr[dev & 63];
}

// A grow-only device buffer kept across calls, for the one large per-level
// scratch whose size climbs level by level (in a bump workspace every larger
// level would strand the previous chunk).  Growing frees the old buffer:
// cudaFree waits for the device, so nothing still reads it.
struct GrowBuf {
  void *p = nullptr;
  size_t cap = 0;
  ~GrowBuf() { if (p) cudaFree(p); }
};
thread_local GrowBuf g_child_scratch_arr[64];
GrowBuf &child_scratch() {
  int d = 0;
  CK(cudaGetDevice(&d));
  return g_child_scratch_arr[d & 63];
}
void *grow_buffer(GrowBuf &b, size_t bytes) {
  if (bytes <= b.cap) return b.p;
  if (b.p) { CK(cudaFree(b.p)); b.p = nullptr; b.cap = 0; }
  const size_t want = bytes + bytes / 4;
  cudaError_t e = cudaMalloc(&b.p, want);
  size_t got = want;
  if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); e = cudaMalloc(&b.p, bytes); got = bytes; }
  if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); b.p = nullptr; throw MrrrError{MRRR_ERR_NOMEM}; }
  CK(e);
  b.cap = got;
  return b.p;
}

// Allocations from one workspace; the workspace is reset when the arena is
// created (a call, a level) -- nothing is freed individually.
struct DevArena {
  BumpWs &ws;
  explicit DevArena(BumpWs &w) : ws(w) { ws.reset(); }
  template <class T>
  T *alloc(size_t count) {
    return (T *)ws.get(count * sizeof(T));
  }
};

// Pinned staging for host->device uploads.  A copy from pageable memory makes
// cudaMemcpyAsync wait for the stream, so every small upload of the
// orchestrator (cluster lists, work items) used to drain the GPU.  Uploads go
// through a per-thread pinned bump buffer instead; a region is never reused
// within a call (mrrr_stemr synchronises its stream before returning, and
// staging_reset() runs at the start of the next call).
struct Staging {
  std::vector<std::pair<char *, size_t>> chunks;  // pinned chunks (kept across calls)
  size_t chunk = 0, off = 0;
  void *get(size_t bytes) {
    bytes = (bytes + 15) & ~size_t(15);
    while (true) {
      if (chunk < chunks.size() && off + bytes <= chunks[chunk].second) {
        void *p = chunks[chunk].first + off;
        off += bytes;
        return p;
      }
      if (chunk + 1 < chunks.size()) { ++chunk; off = 0; continue; }
      size_t sz = std::max<size_t>(bytes, chunks.empty() ? (8u << 20) : 2 * chunks.back().second);
      char *p = nullptr;
      if (cudaMallocHost((void **)&p, sz) != cudaSuccess) { cudaGetLastError(); return nullptr; }
      chunks.push_back({p, sz});
      chunk = chunks.size() - 1;
      off = 0;
    }
  }
  void reset() { chunk = 0; off = 0; }
  ~Staging() {
    for (auto &c : chunks) cudaFreeHost(c.first);
  }
};
thread_local Staging g_staging;

template <class T>
void h2d(T *dst, const T *src, size_t count, cudaStream_t s) {
  if (!count) return;
  void *st = g_staging.get(count * sizeof(T));
  if (st) {
    memcpy(st, src, count * sizeof(T));
    CK(cudaMemcpyAsync(dst, st, count * sizeof(T), cudaMemcpyHostToDevice, s));
  } else {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
}
template <class T>
void d2h(T *dst, const T *src, size_t count, cudaStream_t s) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

// Per-thread event pools, reset at the start of every call (the previous
// call synchronised all its work): no event is created or destroyed per call
// in steady state (driver object churn next to an nvidia-smi sampler cost
// milliseconds per call).
struct EvPool {
  unsigned flags;
  std::vector<cudaEvent_t> ev;
  size_t i = 0;
  ~EvPool() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
  cudaEvent_t get() {
    if (i == ev.size()) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, flags));
      ev.push_back(e);
    }
    return ev[i++];
  }
};
thread_local EvPool g_ev_sync{cudaEventDisableTiming}, g_ev_time{cudaEventDefault};
cudaEvent_t ev_sync() { return g_ev_sync.get(); }
// for destructors (stream joins on every exit path): never throws
void join_streams_nothrow(cudaStream_t waiter, cudaStream_t producer) {
  if (!waiter || !producer || waiter == producer) return;
  try {
    cudaEvent_t e = ev_sync();
    cudaEventRecord(e, producer);
    cudaStreamWaitEvent(waiter, e, 0);
  } catch (...) {
    cudaStreamSynchronize(producer);  // no event available: wait on the host instead
  }
}
cudaEvent_t ev_time() { return g_ev_time.get(); }
void ev_reset() { g_ev_sync.i = 0; g_ev_time.i = 0; }

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    a = ev_time(); b = ev_time(); cudaEventRecord(a, s);
  }
  double stop() {
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    cudaEventRecord(a, s);
    return ms;
  }
};

// Event pair around one group of launches on the call's stream; read at the
// end of the call (no extra synchronisation inside the solve).
struct KTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  bool used = false;
  KTimer() { a = ev_time(); b = ev_time(); }
  void start(cudaStream_t s) { cudaEventRecord(a, s); used = true; }
  void stop(cudaStream_t s) { cudaEventRecord(b, s); }
  double ms() {
    if (!used) return 0.0;
    cudaEventSynchronize(b);
    float v = 0; cudaEventElapsedTime(&v, a, b);
    return v;
  }
};

// Launch helpers -----------------------------------------------------------
__global__ void k_root_interval(const Node *nodes, const Block *blocks, const int *root_nodes,
                                int nroot, double *lo0, double *hi0, double tnrm_scaled, int *fail) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nroot) return;
  const Node N = nodes[root_nodes[r]];
  const Block B = blocks[N.block];
  double sigma = N.tau_hi;
  double wid = 2.0 * kEps * fmax(B.spdiam, tnrm_scaled) + kTiny;
  if (N.nb == 1) { lo0[r] = hi0[r] = __ldg(&N.DL[0]).x; return; }
  bool found = false;
  if (B.side > 0) {
    lo0[r] = 0.0;
    for (int k = 0; k < 200 && !found; ++k) {
      double h = (B.gu - sigma) + wid;
      if ((int)negcount_global(N.DL, N.nb, h, nullptr) >= N.nb) { hi0[r] = h; found = true; }
      wid *= 2.0;
    }
  } else {
    hi0[r] = 0.0;
    for (int k = 0; k < 200 && !found; ++k) {
      double l = (B.gl - sigma) - wid;
      if ((int)negcount_global(N.DL, N.nb, l, nullptr) <= 0) { lo0[r] = l; found = true; }
      wid *= 2.0;
    }
  }
  if (!found) { lo0[r] = hi0[r] = 0.0; fail[0] = 1; }
}

// Warp version: lanes l and l + 16 try the offset wid * 2^(k0 + l % 16) in
// ONE sweep of the root representation, counting as a twisted factorization
// (reading 32, as k_refine_warp): lanes 0-15 the stationary transform over
// rows 0 .. r-1, lanes 16-31 the progressive one over rows nb-2 .. r (the
// bottom tiles copied swapped), half the rows each; the first passing k is
// the sequential loop's answer.
__global__ void __launch_bounds__(32) k_root_interval_warp(const Node *nodes, const Block *blocks,
                                                           const int *root_nodes, int nroot, double *lo0,
                                                           double *hi0, double tnrm_scaled, int *fail) {
  constexpr int T = 16, RING = 6;
  __shared__ double2 ring[RING][2 * T];
  const int r = blockIdx.x, lane = threadIdx.x;
  if (r >= nroot) return;
  const Node N = nodes[root_nodes[r]];
  const Block B = blocks[N.block];
  const double sigma = N.tau_hi;
  const double wid0 = 2.0 * kEps * fmax(B.spdiam, tnrm_scaled) + kTiny;
  if (N.nb == 1) { if (lane == 0) { lo0[r] = hi0[r] = __ldg(&N.DL[0]).x; } return; }
  const int nb = N.nb;
  const bool fwd = lane < 16;
  const int hl = lane & 15;
  const int Lf = ((nb - 1) / (2 * T)) * T, Lb = nb - 1 - Lf;
  const int ntf = Lf / T, ntb = (Lb + T - 1) / T;
  const double Dl = __ldg(&N.DL[nb - 1]).x;
  for (int k0 = 0; k0 < 224; k0 += 16) {
    const double w = wid0 * ldexp(1.0, k0 + hl);
    const double mu = B.side > 0 ? (B.gu - sigma) + w : (B.gl - sigma) - w;
    Sturm st;
    sturm_init(st, mu);
    if (!fwd) st.p = Dl - mu;
    bool ok = true;
    auto issue = [&](int t) {
      if (fwd) {
        if (t < ntf) __pipeline_memcpy_async(&ring[t % RING][hl], &N.DL[t * T + hl], sizeof(double2));
      } else {
        const int row = nb - 2 - (t * T + hl);
        if (t < ntb && row >= Lf) {
          double2 *dst = &ring[t % RING][T + hl];
          __pipeline_memcpy_async(&dst->x, &N.DL[row].y, sizeof(double));
          __pipeline_memcpy_async(&dst->y, &N.DL[row].x, sizeof(double));
        }
      }
      __pipeline_commit();
    };
#pragma unroll
    for (int k = 0; k < RING - 1; ++k) issue(k);
    for (int t = 0; t < ntb; ++t) {
      __pipeline_wait_prior(RING - 2);
      __syncwarp();
      const double2 *TT = ring[t % RING] + (fwd ? 0 : T);
      const int rows = fwd ? (t < ntf ? T : 0) : min(T, Lb - t * T);
      if (rows == T) {
#pragma unroll
        for (int k = 0; k < T; ++k) {
          const double2 v = TT[k];
          sturm_step(st, v.x, v.y, mu);
          if ((k & 7) == 7) ok &= sturm_rescale(st);
        }
      } else {
        for (int k = 0; k < rows; ++k) {
          const double2 v = TT[k];
          sturm_step(st, v.x, v.y, mu);
          if ((k & 7) == 7) ok &= sturm_rescale(st);
        }
      }
      __syncwarp();
      issue(t + RING - 1);
    }
    __pipeline_wait_prior(0);
    ok &= sturm_rescale(st);
    ok &= sturm_ok(st);
    ok &= __shfl_xor_sync(0xffffffffu, (int)ok, 16) != 0;
    const double a = __shfl_xor_sync(0xffffffffu, st.p, 16);
    const double b = __shfl_xor_sync(0xffffffffu, st.q, 16);
    const unsigned cb = __shfl_xor_sync(0xffffffffu, st.c, 16);
    const double X = fma(mu, st.q, st.p);
    const double Ng = fma(X, b, a * st.q);
    unsigned c = st.c + cb + ((Ng != 0.0) ? (((unsigned)(hi32(Ng) ^ hi32(st.q) ^ hi32(b))) >> 31) : 0u);
    if (fwd && (!ok || g_force_safe)) c = negcount_qd_safe(N.DL, nb, mu);
    const bool pass = fwd && (B.side > 0 ? ((int)c >= nb) : ((int)c <= 0));
    const unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (bal) {
      const int first = __ffs(bal) - 1;
      const double m = __shfl_sync(0xffffffffu, mu, first);
      if (lane == 0) {
        if (B.side > 0) { lo0[r] = 0.0; hi0[r] = m; }
        else { hi0[r] = 0.0; lo0[r] = m; }
      }
      return;
    }
  }
  if (lane == 0) { lo0[r] = hi0[r] = 0.0; fail[0] = 1; }  // no enclosing bound within 224 doublings
}

__global__ void k_block_norms(const double *ds, const double *es, Block *blocks, int nblocks) {
  int b = blockIdx.x;
  if (b >= nblocks) return;
  Block B = blocks[b];
  double lo = CUDART_INF, hi = -CUDART_INF;
  for (int i = threadIdx.x; i < B.nb; i += blockDim.x) {
    int64_t g = B.row0 + i;
    double r = 0;
    if (i > 0) r += fabs(es[g - 1]);
    if (i < B.nb - 1) r += fabs(es[g]);
    lo = fmin(lo, ds[g] - r);
    hi = fmax(hi, ds[g] + r);
  }
  __shared__ double sl[32], sh[32];
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffff, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffff, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { sl[threadIdx.x >> 5] = lo; sh[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fmin(lo, sl[w]); hi = fmax(hi, sh[w]); }
    lo = fmin(lo, sl[0]); hi = fmax(hi, sh[0]);
    blocks[b].gl = lo; blocks[b].gu = hi; blocks[b].spdiam = hi - lo;
  }
}

// Root node entries (one per block with members).
__global__ void k_root_nodes(Node *nodes, const Block *blocks, const int *root_blocks, int nroot,
                             const double2 *DLroot, const double *sigma_b) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nroot) return;
  int b = root_blocks[r];
  Block B = blocks[b];
  Node N;
  N.DL = DLroot + B.row0;
  N.row0 = B.row0; N.nb = B.nb; N.block = b;
  N.slot0 = B.slot0; N.slot1 = B.slot1; N.depth = 0; N.jbase = B.jlo;
  N.tau_hi = sigma_b[b]; N.tau_lo = 0.0; N.spdiam = B.spdiam; N.sigma = 0.0;
  N.parent = -1; N.pad = 0;
  nodes[B.root_node] = N;
}

// Child node entries and bracket translation to child coordinates (O9.4).
// cl_rrr[c]: cluster c's child RRR slot on this rank, null when another
// rank owns the cluster (multi-GPU: the entry keeps the tree's numbering; its
// representation is never read here)
__global__ void k_child_nodes(Node *nodes, int node_base, const int *cl_parent, const int *cl_s0,
                              const int *cl_s1, const double *sigma, int ncl, double2 *const *cl_rrr,
                              const int *slot_jlocal) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  Node P = nodes[cl_parent[c]];
  Node N = P;
  N.DL = cl_rrr[c];
  N.slot0 = cl_s0[c]; N.slot1 = cl_s1[c];
  N.depth = P.depth + 1;
  N.jbase = slot_jlocal[cl_s0[c]];
  dd_add(P.tau_hi, P.tau_lo, sigma[c], N.tau_hi, N.tau_lo);
  N.sigma = sigma[c];
  N.parent = cl_parent[c];
  nodes[node_base + c] = N;
}

__global__ void k_translate(const int *slot_cl, const int *cl_first_slot, int nslots_new,
                            const double *sigma, double *lo, double *hi, double *wl, double *wu,
                            int *slot_node, int node_base) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nslots_new) return;
  int c = slot_cl[q];
  int s = cl_first_slot[q];
  double sg = sigma[c];
  double l = lo[s], h = hi[s];
  double lam = 0.5 * (l + h);
  double w = 2.0 * (h - l) + 4.0 * kEps * (fabs(sg) + fabs(lam));
  lo[s] = l - sg; hi[s] = h - sg;
  wl[s] = w; wu[s] = w;
  slot_node[s] = node_base + c;
}

// e: merge of the bracket exchange -- slot q takes the brackets of its
// owner rank (recv holds the ranks' [lo | hi | header] arrays, stride apart)
__global__ void k_merge_brackets(const double *recv, int64_t stride, int nslots, const int *owner, double *lo,
                                 double *hi) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nslots) return;
  const double *src = recv + (int64_t)owner[q] * stride;
  lo[q] = src[q];
  hi[q] = src[nslots + q];
}

__global__ void k_scatter(const int *idx, const double *src, int n, double *dst) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}

__global__ void k_output(const VecTask *tasks, int ntask, const Node *nodes, const double *lam,
                         double inv_scale, double *w) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntask) return;
  const Node N = nodes[tasks[t].node];
  double v = __dadd_rn(N.tau_hi, __dadd_rn(N.tau_lo, lam[t]));
  w[tasks[t].col] = v * inv_scale;
}

__global__ void k_values(const int *slot_node, const int *slot_out, const Node *nodes,
                         const double *lo, const double *hi, int nslots, double inv_scale,
                         double *w) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslots || slot_out[s] < 0) return;
  const Node N = nodes[slot_node[s]];
  double mid = 0.5 * (lo[s] + hi[s]);
  w[slot_out[s]] = __dadd_rn(N.tau_hi, __dadd_rn(N.tau_lo, mid)) * inv_scale;
}

// O11 monotone fix w_j <- max(w_j, w_{j-1}): one CTA, chunked prefix max.
__global__ void k_monotone(double *w, int m) {
  __shared__ double cmax[1024];
  int T = blockDim.x;
  int per = (m + T - 1) / T;
  int a = threadIdx.x * per, b = min(a + per, m);
  double mx = -CUDART_INF;
  for (int i = a; i < b; ++i) mx = fmax(mx, w[i]);
  cmax[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = -CUDART_INF;
    for (int t = 0; t < T; ++t) { double v = cmax[t]; cmax[t] = run; run = fmax(run, v); }
  }
  __syncthreads();
  double run = cmax[threadIdx.x];
  for (int i = a; i < b; ++i) { run = fmax(run, w[i]); w[i] = run; }
}

// Running max + slot assignment for the grid stage (single CTA, chunked).
__global__ void k_grid_assign2(int *cnt, int G, int nb, double lo0, double hi0, const int *slot_j,
                               int s0, int s1, double *lo, double *hi) {
  __shared__ int cm[1024];
  int T = blockDim.x;
  int tot = G + 1;
  int per = (tot + T - 1) / T;
  int a = threadIdx.x * per, b = min(a + per, tot);
  int mx = 0;
  for (int g = a; g < b; ++g) {
    int v = (g == 0) ? 0 : (g == G ? nb : cnt[g]);
    mx = max(mx, v);
  }
  cm[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int t = 0; t < T; ++t) { int v = cm[t]; cm[t] = run; run = max(run, v); }
  }
  __syncthreads();
  int run = cm[threadIdx.x];
  for (int g = a; g < b; ++g) {
    int v = (g == 0) ? 0 : (g == G ? nb : cnt[g]);
    run = max(run, v);
    cnt[g] = run;
  }
  __syncthreads();
  __threadfence_block();
  for (int s = s0 + threadIdx.x; s < s1; s += T) {
    int j = slot_j[s];
    int lo_g = 0, hi_g = G;
    while (lo_g < hi_g) {
      int mid = (lo_g + hi_g) >> 1;
      if (cnt[mid] >= j) hi_g = mid; else lo_g = mid + 1;
    }
    int g = max(lo_g, 1);
    lo[s] = (g - 1 == 0) ? lo0 : lo0 + (hi0 - lo0) * ((double)(g - 1) / (double)G);
    hi[s] = (g == G) ? hi0 : lo0 + (hi0 - lo0) * ((double)g / (double)G);
  }
}

// grid points g in [g_begin, g_end) of the G-interval grid (1 <= g_begin, g_end <= G)
void launch_grid(int M, const Node *nodes, int node, double lo0, double hi0, int G, int g_begin, int g_end,
                 int *cnt, unsigned long long *safe, cudaStream_t s) {
  int pts = g_end - g_begin;
  int per_cta = 128 * M;
  int grid = (pts + per_cta - 1) / per_cta;
  if (grid <= 0) return;
  switch (M) {
    case 1: k_grid<1><<<grid, 128, 0, s>>>(nodes, node, lo0, hi0, G, g_begin, g_end, cnt, safe); break;
    case 2: k_grid<2><<<grid, 128, 0, s>>>(nodes, node, lo0, hi0, G, g_begin, g_end, cnt, safe); break;
    default: k_grid<4><<<grid, 128, 0, s>>>(nodes, node, lo0, hi0, G, g_begin, g_end, cnt, safe); break;
  }
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
}

struct HostNode {
  int slot0, slot1, depth, block;
};

// Warp items: runs of at most 32 consecutive tasks spanning at most maxseg
// nodes of one block (kernels_warp.cuh, kMaxSeg); maxseg = 1 gives one node
// per item (MRRR_VEC_PACK=0, diagnostic: the per-lane arithmetic is the same,
// so the results are bit-identical).
std::vector<WarpItem> make_warp_items(const std::vector<VecTask> &t, const std::vector<HostNode> &hn,
                                      int maxseg, int lanes = 32) {
  std::vector<WarpItem> v;
  const int nt = (int)t.size();
  for (int a = 0; a < nt;) {
    int b = a, segs = 0, prev = -1;
    while (b < nt && b - a < lanes) {
      const int nd = t[b].node;
      if (nd != prev) {
        if (segs == maxseg || (prev >= 0 && hn[nd].block != hn[prev].block)) break;
        ++segs;
        prev = nd;
      }
      ++b;
    }
    WarpItem w; w.node = t[a].node; w.t0 = a; w.t1 = b; w.nsegs = segs;
    v.push_back(w);
    a = b;
  }
  return v;
}

// pair = true: k_wvectors_pair (one item per CTA on two warps, one sweep of
// latency per factorization); false: k_wvectors (one warp per item).
void launch_wvec(WVecArgs A, cudaStream_t s, bool pair) {
  const size_t smem1 = kSingleWarps * sizeof(WarpSmem), smem2 = 2 * sizeof(WarpSmem) + sizeof(PairX);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_wvectors, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
    CK(cudaFuncSetAttribute(k_wvectors_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    attr = true;
  }
  if (A.nitems == 0) return;
  if (pair) k_wvectors_pair<<<A.nitems, kPairThreads, smem2, s>>>(A);
  else k_wvectors<<<(A.nitems + kSingleWarps - 1) / kSingleWarps, 32 * kSingleWarps, smem1, s>>>(A);
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
}

// The split RQC's phases (mode 3: full factorization + first update; mode 4:
// the rest + solve with task_list = the twist-sorted order).
void launch_wsplit(WVecArgs A, int mode, cudaStream_t s) {
  const size_t smem = kSingleWarps * sizeof(WarpSmem);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_wvectors_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (A.nitems == 0) return;
  A.mode = mode;
  k_wvectors_split<<<(A.nitems + kSingleWarps - 1) / kSingleWarps, 32 * kSingleWarps, smem, s>>>(A);
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
}

// The same phases on warp pairs (k_wvectors_psplit).
void launch_wpsplit(WVecArgs A, int mode, cudaStream_t s) {
  const size_t smem2 = 2 * sizeof(WarpSmem) + sizeof(PairX);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_wvectors_psplit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    attr = true;
  }
  if (A.nitems == 0) return;
  A.mode = mode;
  k_wvectors_psplit<<<A.nitems, kPairThreads, smem2, s>>>(A);
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
}

struct SplitBufs {
  RqcState *state;
  int *rkey, *rkey_out, *perm_in, *perm, *seg_b, *seg_e;
  int nseg, bits;
  size_t temp_bytes;
  char *temp;
};

__global__ void k_iota(int *v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// Adaptive multisection by warps (k_refine_warp) over work items of at most
// kRWMembers slots.
void launch_refine(const Node *nodes, const Work *work, int nwork, const int *slot_list,
                   const int *slot_j, double *lo, double *hi, const double *wlo, const double *whi,
                   int verify, double rtol, int *fail, unsigned long long *sweeps,
                   unsigned long long *safe, cudaStream_t s, int M = 4, double class_tol = 0.0,
                   double early_w = 0.0, bool split = false) {
  if (nwork == 0) return;
  const int grid = (nwork + kRWWarps - 1) / kRWWarps;
#define MRRR_RW(MM, SP)                                                                                   \
  k_refine_warp<MM, SP><<<grid, 32 * kRWWarps, 0, s>>>(nodes, work, nwork, slot_list, slot_j, lo, hi, wlo, \
                                                       whi, verify, rtol, 4000, fail, sweeps, safe, class_tol, \
                                                       early_w)
  if (M == 1) {
    if (split) MRRR_RW(1, true); else MRRR_RW(1, false);
  } else if (M == 2) {
    if (split) MRRR_RW(2, true); else MRRR_RW(2, false);
  } else {
    if (split) MRRR_RW(4, true); else MRRR_RW(4, false);
  }
#undef MRRR_RW
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
}

struct Problem {
  int64_t n;
  const double *d, *e;
  int range;
  double vl, vu;
  int64_t il, iu;
  double *w, *Z;
  int64_t ldz;
  cudaStream_t s;
  mrrr_opts_t o;
  // distributed (single GPU: rank 0 of 1); DESIGN.md §6
  int rank = 0, nranks = 1;
  mrrr_allgather_fn allgather = nullptr;
  void *ag_ctx = nullptr;
  double *w_all = nullptr;  // dist: all m eigenvalues (device); P.w is then unused
  int64_t col_begin = 0, m_local = 0;
  // host entry with a pinned destination: Z column blocks are downloaded to
  // hZ (leading dimension hldz) as soon as their vectors are written
  double *hZ = nullptr;
  int64_t hldz = 0;
};


// The solve runs on a library stream of the device's greatest priority,
// ordered after the caller's stream on entry and before it on every exit:
// when the vector pieces (side streams, default priority) and the tree's
// kernels wait for SM resources at the same time, the block scheduler
// serves the tree -- the critical path -- first.
cudaStream_t hp_stream() {
  int d = 0;
  CK(cudaGetDevice(&d));
  cudaStream_t &x = g_streams.st[d & 63][kSide + 1];
  if (!x) {
    int lo_pr = 0, hi_pr = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_pr, &hi_pr));
    CK(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, hi_pr));
  }
  return x;
}

// A second high-priority stream for the tree: the interior-candidate step
// of the big clusters (reading 30) runs beside the other clusters' step.
cudaStream_t hp_stream2() {
  int d = 0;
  CK(cudaGetDevice(&d));
  cudaStream_t &x = g_streams.st[d & 63][kSide + 2];
  if (!x) {
    int lo_pr = 0, hi_pr = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_pr, &hi_pr));
    CK(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, hi_pr));
  }
  return x;
}

// e: shard planner.  cuts[0..nranks] start as the static division (rank r
// owns columns [cuts[r], cuts[r+1])); each inner cut moves to the nearest
// column j with free_cut[j] != 0 (a cluster boundary between columns j-1
// and j) within epp / 40, so a share grows by at most epp / 20 (5 %).  Ties
// go to the left.  Deterministic: every rank computes the same cuts.
void plan_columns(int64_t m, int nranks, const unsigned char *free_cut, int64_t *cuts) {
  const int64_t epp = (m + nranks - 1) / nranks, slack = epp / 40;
  for (int r = 0; r <= nranks; ++r) cuts[r] = std::min<int64_t>((int64_t)r * epp, m);
  for (int r = 1; r < nranks; ++r) {
    const int64_t t = cuts[r];
    if (t <= cuts[r - 1] || t >= m) { cuts[r] = std::max(cuts[r - 1], std::min(t, m)); continue; }
    int64_t best = -1;
    for (int64_t d = 0; d <= slack && best < 0; ++d) {
      if (t - d > cuts[r - 1] && t - d > 0 && free_cut[t - d]) best = t - d;
      else if (t + d < m && free_cut[t + d]) best = t + d;
    }
    if (best >= 0) cuts[r] = best;
  }
}

// Diagnostic switches of common.cuh from the environment (tests only),
// written to the device only when they change.
void set_diag_flags(cudaStream_t s) {
  static int last_safe[64], last_nudge[64];
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const int fs = env_int("MRRR_FORCE_SAFE", 0) != 0, fn = env_int("MRRR_FORCE_NUDGE", 0) != 0;
  if (fs != last_safe[dev & 63]) {
    CK(cudaMemcpyToSymbolAsync(g_force_safe, &fs, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    last_safe[dev & 63] = fs;
  }
  {
    // diagnostic: MRRR_RQC_PREV_TOL=<x> sets the previous-correction stop of the RQC (reading 33; 0 = off)
    static double last_pt[64];
    static bool have_pt[64];
    const char *ev = getenv("MRRR_RQC_PREV_TOL");
    const double pt = ev ? atof(ev) : 4.656612873077393e-10;
    if (!have_pt[dev & 63] ? ev != nullptr : pt != last_pt[dev & 63]) {
      CK(cudaMemcpyToSymbolAsync(g_rqc_prev_tol, &pt, sizeof(double), 0, cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));
    }
    have_pt[dev & 63] = true;
    last_pt[dev & 63] = pt;
  }
  {
    static int last_dbg[64];
    const int fd = env_int("MRRR_DEBUG_RQC", 0);
    if (fd != last_dbg[dev & 63]) {
      CK(cudaMemcpyToSymbolAsync(g_debug_rqc, &fd, sizeof(int), 0, cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));
      last_dbg[dev & 63] = fd;
    }
  }
  if (fn != last_nudge[dev & 63]) {
    CK(cudaMemcpyToSymbolAsync(g_force_nudge, &fn, sizeof(int), 0, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    last_nudge[dev & 63] = fn;
  }
}

int solve(Problem &P, int64_t *m_out) {
  ev_reset();
  const int use_hp = env_int("MRRR_HP_STREAM", 1);
  cudaStream_t s = use_hp ? hp_stream() : P.s;
  set_diag_flags(P.s);
  struct Join {  // caller's stream waits for the solve stream on every exit
    cudaStream_t user, inner;
    ~Join() { join_streams_nothrow(user, inner); }
  } join{P.s, s};
  if (s != P.s) {
    cudaEvent_t e = ev_sync();
    CK(cudaEventRecord(e, P.s));
    CK(cudaStreamWaitEvent(s, e, 0));
  }
  const int64_t n = P.n;
  DevArena ar(device_ws(g_ws_call));
  device_ws(g_ws_level).used_peak = 0;
  size_t cs_scratch_used = 0;
  Trace tr;
  g_staging.reset();
  Timer tm(s), tall(s);
  // MRRR_TIMELINE=1 (diagnostic): device timestamps of the tree's steps and
  // of every vector piece, printed after the solve (no synchronisation in
  // between, unlike MRRR_TRACE=2)
  const bool timeline = getenv("MRRR_TIMELINE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tline;
  std::vector<double> tline_host;  // host clock when the mark was enqueued (ms since the call began)
  const auto tl_host0 = std::chrono::steady_clock::now();
  int tl_level = -1;
  auto tl_mark = [&](const std::string &what) {
    if (!timeline) return;
    cudaEvent_t e = ev_time();
    cudaEventRecord(e, s);
    tline.push_back({what, e});
    tline_host.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl_host0).count());
  };
  KTimer kt_root, kt_fin;
  memset(&g_stats, 0, sizeof(g_stats));
  memset(g_rqc_hist, 0, sizeof(g_rqc_hist));
  const bool vectors = P.Z != nullptr;

  // ---------------- a1: prep ----------------
  tr.phase("mrrr root");
  double *ds = ar.alloc<double>(n), *es = ar.alloc<double>(n), *es2 = ar.alloc<double>(n);
  int *brk = ar.alloc<int>(n);
  double *hdr = ar.alloc<double>(8);
  unsigned long long *ctr = ar.alloc<unsigned long long>(48);  // [32..47]: the RQC histogram
  CK(cudaMemsetAsync(ctr, 0, 48 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(brk, 0, n * sizeof(int), s));
  k_prep<<<1, 1024, 0, s>>>(P.d, P.e, n, ds, es, es2, brk, hdr);
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
  double h_hdr[5];
  d2h(h_hdr, hdr, 5, s);
  if (h_hdr[4] == 1.0) throw MrrrError{-2};  // non-finite d
  if (h_hdr[4] == 2.0) throw MrrrError{-3};  // non-finite e
  const double scale = h_hdr[1];
  const double tnrm_s = h_hdr[0] * scale;
  std::vector<int> h_brk(n);
  d2h(h_brk.data(), brk, n, s);
  tr.mark("prep");

  // blocks
  std::vector<Block> hb;
  {
    int64_t st = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (i == n - 1 || h_brk[i]) {
        Block B{};
        B.row0 = st; B.nb = (int)(i - st + 1);
        hb.push_back(B);
        st = i + 1;
      }
    }
  }
  const int nblocks = (int)hb.size();
  Block *dblocks = ar.alloc<Block>(nblocks);
  h2d(dblocks, hb.data(), nblocks, s);
  k_block_norms<<<nblocks, 256, 0, s>>>(ds, es, dblocks, nblocks);
  CK(cudaGetLastError());
  g_stats.kernel_launches++;
  d2h(hb.data(), dblocks, nblocks, s);

  // ---------------- O4: wanted ranges per block ----------------
  std::vector<int> wa(nblocks), wb(nblocks);
  auto sturm_counts = [&](const std::vector<double> &xs) {
    // counts[x][block] on the scaled split T
    double *dx = ar.alloc<double>(xs.size());
    int *dc = ar.alloc<int>(xs.size() * nblocks);
    h2d(dx, xs.data(), xs.size(), s);
    int tot = (int)xs.size() * nblocks;
    k_sturm_T<<<(tot + 127) / 128, 128, 0, s>>>(ds, es2, dblocks, nblocks, dx, (int)xs.size(), dc);
    CK(cudaGetLastError());
    g_stats.kernel_launches++;
    std::vector<int> hc(tot);
    d2h(hc.data(), dc, tot, s);
    return hc;
  };
  int64_t base_rank = 0;
  bool multi_index = false;
  if (P.range == MRRR_RANGE_ALL) {
    for (int b = 0; b < nblocks; ++b) { wa[b] = 1; wb[b] = hb[b].nb; }
  } else if (P.range == MRRR_RANGE_VALUE) {
    auto c = sturm_counts({P.vl * scale, P.vu * scale});
    for (int b = 0; b < nblocks; ++b) { wa[b] = c[b] + 1; wb[b] = c[nblocks + b]; }
  } else if (nblocks == 1) {
    wa[0] = (int)P.il; wb[0] = (int)P.iu;
  } else {
    // brackets of the il-th and iu-th eigenvalue of the split matrix by
    // multisection on T's Sturm counts (64 shifts per round)
    multi_index = true;
    double glo = INFINITY, ghi = -INFINITY;
    for (auto &B : hb) { glo = std::min(glo, B.gl); ghi = std::max(ghi, B.gu); }
    double wid = 4.0 * kEps * tnrm_s;
    auto bracket = [&](int64_t idx, bool want_lo) {
      double a = glo - 2 * wid - kTiny, b = ghi + 2 * wid + kTiny;
      for (int it = 0; it < 40 && b - a > wid; ++it) {
        std::vector<double> xs(63);
        for (int k = 0; k < 63; ++k) xs[k] = a + (b - a) * ((k + 1) / 64.0);
        auto c = sturm_counts(xs);
        double na = a, nbb = b;
        for (int k = 0; k < 63; ++k) {
          int64_t tot = 0;
          for (int bb = 0; bb < nblocks; ++bb) tot += c[k * nblocks + bb];
          if (tot < idx) na = std::max(na, xs[k]);
        }
        for (int k = 62; k >= 0; --k) {
          int64_t tot = 0;
          for (int bb = 0; bb < nblocks; ++bb) tot += c[k * nblocks + bb];
          if (tot >= idx && xs[k] > na) nbb = std::min(nbb, xs[k]);
        }
        a = na; b = nbb;
      }
      return want_lo ? a : b;
    };
    double xa = bracket(P.il, true), xb = bracket(P.iu, false);
    auto c = sturm_counts({xa, xb});
    for (int b = 0; b < nblocks; ++b) {
      wa[b] = c[b] + 1; wb[b] = c[nblocks + b];
      base_rank += c[b];
    }
  }

  // members per block: wanted range plus gap neighbours (reading 7)
  std::vector<int> ma(nblocks), mb(nblocks);
  int64_t nslots = 0;
  for (int b = 0; b < nblocks; ++b) {
    if (wb[b] < wa[b]) { ma[b] = 1; mb[b] = 0; continue; }
    ma[b] = std::max(1, wa[b] - 1);
    mb[b] = std::min(hb[b].nb, wb[b] + 1);
    if (nblocks > 1 && !vectors) { ma[b] = wa[b]; mb[b] = wb[b]; }
    nslots += mb[b] - ma[b] + 1;
  }
  std::vector<int> h_slot_j(nslots), h_slot_block(nslots), h_slot_out(nslots, -1);
  std::vector<int> root_blocks;
  int nnodes = 0;
  {
    int64_t q = 0;
    for (int b = 0; b < nblocks; ++b) {
      hb[b].slot0 = (int)q;
      for (int j = ma[b]; j <= mb[b]; ++j) { h_slot_j[q] = j; h_slot_block[q] = b; ++q; }
      hb[b].slot1 = (int)q;
      hb[b].jlo = ma[b];
      hb[b].side = (wa[b] + wb[b] <= hb[b].nb + 1) ? 1 : -1;
      hb[b].root_node = -1;
      if (hb[b].slot1 > hb[b].slot0) { hb[b].root_node = nnodes++; root_blocks.push_back(b); }
    }
  }
  const int nroot = (int)root_blocks.size();
  int64_t m = 0;
  if (nroot == 0) { *m_out = 0; return 0; }
  h2d(dblocks, hb.data(), nblocks, s);

  // ---------------- a2: root representations ----------------
  double2 *DLroot = ar.alloc<double2>(n), *LDv = ar.alloc<double2>(n);
  double *tbuf = ar.alloc<double>(n);
  int *sbuf = ar.alloc<int>(n);
  double *sigma_b = ar.alloc<double>(nblocks);
  int *dfail = ar.alloc<int>(4);
  CK(cudaMemsetAsync(dfail, 0, 4 * sizeof(int), s));
  CK(cudaMemsetAsync(sigma_b, 0, nblocks * sizeof(double), s));
  if (nblocks <= 4096)  // one warp per block (smem-tiled chain); many tiny blocks: one thread each
    k_root_chain_warp<<<nblocks, 32, 0, s>>>(ds, es2, dblocks, nblocks, tnrm_s, tbuf, sbuf, sigma_b, dfail);
  else
    k_root_chain<<<(nblocks + 63) / 64, 64, 0, s>>>(ds, es2, dblocks, nblocks, tnrm_s, tbuf, sbuf,
                                                    sigma_b, dfail);
  CK(cudaGetLastError());
  std::vector<int> h_row_block(n);
  for (int b = 0; b < nblocks; ++b)
    for (int i = 0; i < hb[b].nb; ++i) h_row_block[hb[b].row0 + i] = b;
  int *row_block = ar.alloc<int>(n);
  h2d(row_block, h_row_block.data(), n, s);
  k_root_finish<<<(n + 255) / 256, 256, 0, s>>>(ds, es, dblocks, row_block, n, tbuf, sbuf, sigma_b,
                                                P.o.perturb_root, P.o.seed, DLroot, LDv);
  CK(cudaGetLastError());
  g_stats.kernel_launches += 2;
  int h_fail[4];
  d2h(h_fail, dfail, 4, s);
  if (h_fail[0]) throw MrrrError{MRRR_ERR_ROOT};
  dump("root_DL.bin", DLroot, n, s);
  dump("root_LDv.bin", LDv, n, s);
  dump("root_sigma.bin", sigma_b, nblocks, s);
  tr.mark("root rrr");

  // node table (device), capacity grows with levels
  int node_cap = std::max<int>(nroot + 16, 64);
  Node *dnodes = ar.alloc<Node>(node_cap);
  std::vector<int> h_root_blocks(root_blocks);
  int *droot_blocks = ar.alloc<int>(nroot);
  h2d(droot_blocks, h_root_blocks.data(), nroot, s);
  k_root_nodes<<<(nroot + 63) / 64, 64, 0, s>>>(dnodes, dblocks, droot_blocks, nroot, DLroot,
                                                  sigma_b);
  CK(cudaGetLastError());
  std::vector<int> h_root_nodes(nroot);
  for (int r = 0; r < nroot; ++r) h_root_nodes[r] = hb[root_blocks[r]].root_node;
  int *droot_nodes = ar.alloc<int>(nroot);
  h2d(droot_nodes, h_root_nodes.data(), nroot, s);
  double *dlo0 = ar.alloc<double>(nroot), *dhi0 = ar.alloc<double>(nroot);
  if (nroot <= 4096)
    k_root_interval_warp<<<nroot, 32, 0, s>>>(dnodes, dblocks, droot_nodes, nroot, dlo0, dhi0, tnrm_s, dfail + 3);
  else
    k_root_interval<<<(nroot + 63) / 64, 64, 0, s>>>(dnodes, dblocks, droot_nodes, nroot, dlo0, dhi0,
                                                     tnrm_s, dfail + 3);
  CK(cudaGetLastError());
  g_stats.kernel_launches += 2;
  std::vector<double> hlo0(nroot), hhi0(nroot);
  d2h(hlo0.data(), dlo0, nroot, s);
  d2h(hhi0.data(), dhi0, nroot, s);
  {
    int hf[4];
    d2h(hf, dfail, 4, s);
    if (hf[3]) throw MrrrError{MRRR_ERR_CONVERGE};  // no root interval found
  }

  // slots (device).  slo and shi are the two halves of one array whose tail
  // holds the exchange header of a multi-GPU rank (status, clusters): one
  // all-gather moves a rank's brackets and header together.
  int *slot_j = ar.alloc<int>(nslots), *slot_node = ar.alloc<int>(nslots);
  int *slot_out = ar.alloc<int>(nslots);
  const int64_t xstride = 2 * nslots + 2;  // doubles per rank in the bracket exchange
  double *slo = ar.alloc<double>(xstride);
  double *shi = slo + nslots, *xhdr = slo + 2 * nslots;
  std::vector<int> h_slot_node(nslots);
  std::vector<double> h_lo(nslots), h_hi(nslots);
  for (int r = 0; r < nroot; ++r) {
    const Block &B = hb[root_blocks[r]];
    for (int q = B.slot0; q < B.slot1; ++q) {
      h_slot_node[q] = B.root_node; h_lo[q] = hlo0[r]; h_hi[q] = hhi0[r];
    }
  }
  h2d(slot_j, h_slot_j.data(), nslots, s);
  h2d(slot_node, h_slot_node.data(), nslots, s);
  h2d(slo, h_lo.data(), nslots, s);
  h2d(shi, h_hi.data(), nslots, s);

  // ---- e: the ranks' collectives.  Every rank calls the same
  // sequence of all-gathers; each carries a status word so that an error on
  // one rank stops all of them at the same exchange (no rank is left waiting).
  const int nr = std::max(1, P.nranks);
  const bool dist = nr > 1;
  // cap of each of the two large scratch areas (vector checkpoints, cluster
  // step scratch): opts.scratch_gb (16 by default); MRRR_SCRATCH_GB overrides
  // (virtual ranks sharing one GPU), MRRR_CK_GB / MRRR_CS_GB one of the two
  // (diagnostic)
  const double scratch_gb = getenv("MRRR_SCRATCH_GB") ? std::max(0.25, atof(getenv("MRRR_SCRATCH_GB")))
                            : P.o.scratch_gb > 0 ? P.o.scratch_gb : 16.0;
  const double ck_bytes = 1e9 * (getenv("MRRR_CK_GB") ? std::max(0.25, atof(getenv("MRRR_CK_GB"))) : scratch_gb);
  const double scratch_bytes = 1e9 * (getenv("MRRR_CS_GB") ? std::max(0.25, atof(getenv("MRRR_CS_GB"))) : scratch_gb);
  double *xrecv = dist ? ar.alloc<double>((size_t)nr * xstride) : nullptr;
  int *slot_owner = dist ? ar.alloc<int>(nslots) : nullptr;
  std::vector<int> h_slot_owner(dist ? nslots : 0, 0);
  int local_status = 0;
  // all-gather of this rank's brackets (+ header) and merge: each slot takes
  // the brackets of the rank that owns it (h_slot_owner); returns the
  // maximum over the ranks of header word 1 and throws the worst status
  auto exchange_brackets = [&](double hdr1) -> double {
    double hh[2] = {(double)local_status, hdr1};
    h2d(xhdr, hh, 2, s);
    if (P.allgather(P.ag_ctx, slo, xrecv, (size_t)xstride * sizeof(double), (void *)s) != 0)
      throw MrrrError{MRRR_ERR_COMM};
    h2d(slot_owner, h_slot_owner.data(), nslots, s);
    k_merge_brackets<<<(int)((nslots + 255) / 256), 256, 0, s>>>(xrecv, xstride, (int)nslots, slot_owner, slo, shi);
    CK(cudaGetLastError());
    g_stats.kernel_launches++;
    std::vector<double> hdrs(2 * (size_t)nr);
    for (int r = 0; r < nr; ++r) CK(cudaMemcpyAsync(&hdrs[2 * r], xrecv + (int64_t)r * xstride + 2 * nslots,
                                                    2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int worst = 0;
    double mx = 0;
    for (int r = 0; r < nr; ++r) {
      const int st = (int)hdrs[2 * r];
      if (st != 0 && (worst == 0 || st > worst)) worst = st;
      mx = std::max(mx, hdrs[2 * r + 1]);
    }
    if (worst) throw MrrrError{worst};
    return mx;
  };

  // dist: a failure between two collectives is recorded in local_status and
  // the rank goes on to the next collective, whose status words make every
  // rank leave there with the worst code (one GPU: errors propagate at once)
  auto guarded = [&](auto &&f) {
    if (!dist) { f(); return; }
    try {
      if (local_status == 0) f();
    } catch (const MrrrError &er) {
      if (!local_status) local_status = er.code;
    } catch (const CudaError &ce) {
      cudaGetLastError();
      if (!local_status) local_status = ce.e == cudaErrorMemoryAllocation ? MRRR_ERR_NOMEM : MRRR_ERR_CUDA;
    }
  };

  // ---------------- a3: root eigenvalue intervals ----------------
  const double rtol_root = (vectors && nblocks == 1) ? P.o.rtol_class : 4.0 * kEps;
  const int M = std::max(1, P.o.multisection);
  // Work items of <= wmax member slots of one node.  wmax shrinks when the
  // level has few slots, so that more CTAs (and more shifts per member, i.e.
  // fewer rounds) cover the GPU.
  auto make_work = [&](int node, int s0, int s1, int wmax, std::vector<Work> &wv) {
    for (int a = s0; a < s1; a += wmax) {
      Work W; W.node = node; W.s0 = a; W.s1 = std::min(a + wmax, s1); W.pad = 0;
      wv.push_back(W);
    }
  };
  // members per refinement warp for a node/cluster of m members: a large
  // block is packed 16 to a warp (with M = 2: 4 shifts each while all are
  // active, i.e. near-bisection work per bit), a small one spread thin (up
  // to 64 shifts each, fewer rounds).  Depends on m alone, so every rank that holds a
  // shared cluster forms the same work items (§8(e)).
  // diagnostics (read per call): MRRR_RW_CHUNK / MRRR_RW_M override the refinement work items
  const int rw_env = env_int("MRRR_RW_CHUNK", 0);
  const int rw_m_env = env_int("MRRR_RW_M", 0);
  auto rw_chunk = [&](int m) {
    if (rw_env > 0) return std::min(rw_env, kRWMembers);
    return m >= 128 ? 16 : 8;
  };
  auto rw_chunk_tree = [&](int m) {
    if (rw_env > 0) return std::min(rw_env, kRWMembers);
    (void)m;
    return 8;
  };
  const int rw_m_tree = rw_m_env > 0 ? rw_m_env : 1;
  // shifts per lane of the root refinement (diagnostic MRRR_RW_ROOT_M)
  // (measured, random n=20000: chunks of 16 members with M = 2 -- 1250 warps
  // of four chains each, split counts -- root 5.05 -> 4.3 ms with the grid at
  // one shift per thread, against 625 warps of chunk 32 with M = 4)
  const int rw_m_root = std::max(1, std::min(4, env_int("MRRR_RW_ROOT_M", 2)));
  // reading 31: tree members stop refining at 2^-early_bits once their
  // classification is decided (MRRR_EARLY_BITS; 0 = off, refine all to rtol_class);
  // 2^-7 since the RQC stop of reading 33 (sweep: profiles/r02/setG/r2G_early_bits_sweep.txt)
  const int early_bits = env_int("MRRR_EARLY_BITS", 7);
  // twisted (split) counts in the refinement sweeps (reading 32): 1 = tree
  // levels, 2 = tree and root, 0 = whole stationary sweeps everywhere
  const int split_env = env_int("MRRR_SPLIT", 2);
  const bool split_tree = split_env >= 1, split_root = split_env >= 2;
  // shifts per thread of the root grid (MRRR_GRID_M, diagnostic: 1, 2 or 4)
  const int grid_m = env_int("MRRR_GRID_M", 1);
  // clusters of at least rw_end members refine their two end members in
  // work items of their own (0: off); MRRR_RW_END overrides
  const int rw_end = env_int("MRRR_RW_END", 0);
  // reading 30: weighted-growth bound of the interior candidate (x spdiam);
  // MRRR_INT_WG overrides (diagnostic)
  const double int_wg = getenv("MRRR_INT_WG") ? atof(getenv("MRRR_INT_WG")) : 4.0;
  // the cluster step: one warp per chain (k_child_step: the shortest chain
  // latency, for levels of at most kChildV1Max clusters) or the chains packed
  // into the lanes of three warps (k_child_step2: fewer instructions, for the
  // wide, issue-bound levels); the same arithmetic, bit for bit.
  // MRRR_CHILD_V1 = 1 / 0 forces one of them (diagnostic).
  const int child_v1_env = env_int("MRRR_CHILD_V1", -1);
  // the wide levels' chains lane-dense (k_child_chains3 + k_child_step2<0,
  // true>); MRRR_CHILD_V3=0: k_child_step2 alone (diagnostic)
  const int child_v3_env = env_int("MRRR_CHILD_V3", 1);
  const int c3_groups = std::min(3, std::max(1, env_int("MRRR_C3_GROUPS", 1)));  // clusters per chain warp
  constexpr int kChildV1Max = 296;  // two clusters per SM
  {
    std::vector<Work> wv;
    kt_root.start(s);
    for (int r = 0; r < nroot; ++r) {
      const Block &B = hb[root_blocks[r]];
      int nsl = B.slot1 - B.slot0;
      const int gf = env_int("MRRR_GRID_FACTOR", P.o.grid_factor);  // diagnostic override
      if (nroot == 1 && gf > 0 && nsl >= 64) {
        int G = (int)std::min<int64_t>((int64_t)gf * nsl + 1, 1 << 20);
        G = std::max(G, 256);
        if (!dist) {
          int *cnt = ar.alloc<int>(G + 1);
          launch_grid(grid_m, dnodes, B.root_node, hlo0[r], hhi0[r], G, 1, G, cnt, ctr + 1, s);
          g_stats.root_sweeps += G - 1;
          k_grid_assign2<<<1, 1024, 0, s>>>(cnt, G, B.nb, hlo0[r], hhi0[r], slot_j, B.slot0,
                                            B.slot1, slo, shi);
        } else {
          // e: each rank counts its share gp of the G-1 grid points, one
          // all-gather assembles the counts (the static
          // division of the bisection work, then a gather)
          const int gp = (G - 1 + nr - 1) / nr;
          const int g_lo = 1 + P.rank * gp, g_hi = std::min(G, g_lo + gp);
          int *cnt_part = ar.alloc<int>((size_t)gp + G + 1);
          int *cnt = ar.alloc<int>((size_t)nr * gp + 2);
          guarded([&] {
            if (g_hi > g_lo) launch_grid(grid_m, dnodes, B.root_node, hlo0[r], hhi0[r], G, g_lo, g_hi, cnt_part, ctr + 1, s);
          });
          g_stats.root_sweeps += std::max(0, g_hi - g_lo);
          if (P.allgather(P.ag_ctx, cnt_part + g_lo, cnt + 1, (size_t)gp * sizeof(int), (void *)s) != 0)
            throw MrrrError{MRRR_ERR_COMM};
          k_grid_assign2<<<1, 1024, 0, s>>>(cnt, G, B.nb, hlo0[r], hhi0[r], slot_j, B.slot0,
                                            B.slot1, slo, shi);
        }
        CK(cudaGetLastError());
        g_stats.kernel_launches++;
      }
      make_work(B.root_node, B.slot0, B.slot1, env_int("MRRR_RW_ROOT_CHUNK", 0) > 0 ? std::min(env_int("MRRR_RW_ROOT_CHUNK", 0), kRWMembers) : rw_chunk(B.nb), wv);  // rank-invariant (block size)
    }
    // e: the work items are split into nr contiguous shares; a slot is owned
    // by the rank whose share holds its item, and one all-gather + merge
    // gives every rank all root brackets
    size_t w0 = 0, w1 = wv.size();
    if (dist) {
      const size_t per = (wv.size() + nr - 1) / nr;
      w0 = std::min(wv.size(), (size_t)P.rank * per);
      w1 = std::min(wv.size(), w0 + per);
      for (size_t i = 0; i < wv.size(); ++i)
        for (int q = wv[i].s0; q < wv[i].s1; ++q) h_slot_owner[q] = (int)(i / per);
    }
    Work *dwork = ar.alloc<Work>(std::max<size_t>(wv.size(), 1));
    h2d(dwork, wv.data(), wv.size(), s);
    guarded([&] {
      if (tr.lvl >= 2) {
        unsigned z[64] = {};
        CK(cudaMemcpyToSymbol(g_rw_hist, z, sizeof z));
      }
      launch_refine(dnodes, dwork + w0, (int)(w1 - w0), nullptr, slot_j, slo, shi, nullptr, nullptr, 0, rtol_root,
                    dfail + 2, ctr, ctr + 1, s, rw_m_root, 0.0, 0.0, split_root);
      if (tr.lvl >= 2) {  // diagnostic: rounds per root refinement warp
        CK(cudaStreamSynchronize(s));
        unsigned hist[64];
        CK(cudaMemcpyFromSymbol(hist, g_rw_hist, sizeof hist));
        fprintf(stderr, "[mrrr]   root refine: %d items; rounds histogram:", (int)(w1 - w0));
        for (int r = 0; r < 64; ++r)
          if (hist[r]) fprintf(stderr, " %d:%u", r, hist[r]);
        fprintf(stderr, "\n");
      }
      if (dist) {
        int hf = 0;
        d2h(&hf, dfail + 2, 1, s);
        if (hf) throw MrrrError{MRRR_ERR_CONVERGE};
      }
    });
    if (dist) exchange_brackets(0.0);
    (void)M;
    kt_root.stop(s);
  }
  {
    int hf[4];
    d2h(hf, dfail, 4, s);
    if (hf[2]) throw MrrrError{MRRR_ERR_CONVERGE};  // root bisection did not converge
  }

  // output positions
  if (nblocks == 1) {
    const Block &B = hb[0];
    for (int q = B.slot0; q < B.slot1; ++q) {
      int j = h_slot_j[q];
      if (j >= wa[0] && j <= wb[0]) h_slot_out[q] = j - wa[0];
    }
    m = wb[0] - wa[0] + 1;
  } else {
    // several blocks: merge by (value, block, index) on the bisected values
    std::vector<double> hv_lo(nslots), hv_hi(nslots);
    d2h(hv_lo.data(), slo, nslots, s);
    d2h(hv_hi.data(), shi, nslots, s);
    std::vector<double> sig(nblocks);
    d2h(sig.data(), sigma_b, nblocks, s);
    struct C { double v; int b, j, q; };
    std::vector<C> cand;
    for (int b = 0; b < nblocks; ++b) {
      if (hb[b].slot1 <= hb[b].slot0) continue;
      double prev = -INFINITY;
      for (int q = hb[b].slot0; q < hb[b].slot1; ++q) {
        int j = h_slot_j[q];
        if (j < wa[b] || j > wb[b]) continue;
        double v = (hb[b].nb == 1) ? 0.0 : sig[b] + 0.5 * (hv_lo[q] + hv_hi[q]);
        if (hb[b].nb == 1) v = 0;  // set below
        cand.push_back({v, b, j, q});
      }
      (void)prev;
    }
    // 1x1 blocks: value is the diagonal entry
    {
      std::vector<double> hds;
      bool need = false;
      for (auto &c : cand) if (hb[c.b].nb == 1) need = true;
      if (need) {
        hds.resize(n);
        d2h(hds.data(), ds, n, s);
        for (auto &c : cand) if (hb[c.b].nb == 1) c.v = hds[hb[c.b].row0];
      }
    }
    // monotone within a block
    for (size_t i = 1; i < cand.size(); ++i)
      if (cand[i].b == cand[i - 1].b && cand[i].v < cand[i - 1].v) cand[i].v = cand[i - 1].v;
    std::vector<int> ord(cand.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
      if (cand[x].v != cand[y].v) return cand[x].v < cand[y].v;
      if (cand[x].b != cand[y].b) return cand[x].b < cand[y].b;
      return cand[x].j < cand[y].j;
    });
    int64_t cnt = 0;
    for (size_t i = 0; i < ord.size(); ++i) {
      const C &c = cand[ord[i]];
      int64_t rank = base_rank + (int64_t)i + 1;
      if (multi_index && (rank < P.il || rank > P.iu)) continue;
      h_slot_out[c.q] = (int)cnt++;
    }
    m = cnt;
  }
  // ---- e: this rank's columns.  The static division of the m wanted pairs
  // (epp = ceil(m / P) per rank); with vectors and one block,
  // the root classification then moves each cut to the nearest cluster
  // boundary within epp / 20 (plan_columns, below), so fewer clusters are
  // shared between ranks.  Every rank builds the same root, intervals and
  // tree structure, works on the clusters its columns touch, and computes
  // only its own vectors.
  const int64_t epp = (m + nr - 1) / nr;
  std::vector<int64_t> cuts(nr + 1);
  for (int r = 0; r <= nr; ++r) cuts[r] = std::min<int64_t>((int64_t)r * epp, m);
  std::vector<int> h_own(nslots, -1);  // local output column of a slot, or -1
  std::vector<int> col_slot(m, -1);    // slot of each output column
  for (int64_t q = 0; q < nslots; ++q)
    if (h_slot_out[q] >= 0) col_slot[h_slot_out[q]] = (int)q;
  auto apply_cuts = [&]() {
    const int64_t c0 = cuts[P.rank], c1 = cuts[P.rank + 1];
    P.col_begin = c0;
    P.m_local = c1 - c0;
    for (int64_t q = 0; q < nslots; ++q)
      h_own[q] = (h_slot_out[q] >= c0 && h_slot_out[q] < c1) ? (int)(h_slot_out[q] - c0) : -1;
    if (!dist) return;
    // slot owners for the bracket exchanges of the tree: the rank of the
    // slot's column; a gap neighbour (no column) goes to the rank of the
    // nearest column of its block
    std::vector<int> col_rank(m);
    for (int r = 0; r < nr; ++r)
      for (int64_t c = cuts[r]; c < cuts[r + 1]; ++c) col_rank[c] = r;
    for (int64_t q = 0; q < nslots; ++q) {
      if (h_slot_out[q] >= 0) { h_slot_owner[q] = col_rank[h_slot_out[q]]; continue; }
      int own = 0;
      for (int64_t d = 1; d < nslots; ++d) {
        if (q - d >= 0 && h_slot_block[q - d] == h_slot_block[q] && h_slot_out[q - d] >= 0) { own = col_rank[h_slot_out[q - d]]; break; }
        if (q + d < nslots && h_slot_block[q + d] == h_slot_block[q] && h_slot_out[q + d] >= 0) { own = col_rank[h_slot_out[q + d]]; break; }
        if (q - d < 0 && q + d >= nslots) break;
      }
      h_slot_owner[q] = own;
    }
  };
  apply_cuts();
  // local eigenvalue buffer: the caller's w on one GPU, a padded buffer of
  // the largest possible share (epp + epp / 20, the planner's slack) for the
  // all-gather otherwise
  const int64_t wcap = std::max<int64_t>(epp + epp / 20, 1);
  double *w_loc = P.w;
  if (nr > 1) {
    w_loc = ar.alloc<double>(wcap + 1);
    CK(cudaMemsetAsync(w_loc, 0, (wcap + 1) * sizeof(double), s));
  }
  // final w: all-gather of the padded local parts (dist; the last word is
  // the rank's status) and the O11 monotone fix
  auto finish_w = [&]() {
    if (nr == 1) {
      if (m > 1) { k_monotone<<<1, 1024, 0, s>>>(P.w, (int)m); CK(cudaGetLastError()); g_stats.kernel_launches++; }
      return;
    }
    double *wall = ar.alloc<double>((size_t)nr * (wcap + 1));
    const double st = (double)local_status;
    h2d(w_loc + wcap, &st, 1, s);
    if (P.allgather(P.ag_ctx, w_loc, wall, (size_t)(wcap + 1) * sizeof(double), (void *)s) != 0)
      throw MrrrError{MRRR_ERR_COMM};
    for (int r = 0; r < nr; ++r)
      if (cuts[r + 1] > cuts[r])
        CK(cudaMemcpyAsync(P.w_all + cuts[r], wall + (int64_t)r * (wcap + 1), (cuts[r + 1] - cuts[r]) * sizeof(double),
                           cudaMemcpyDeviceToDevice, s));
    std::vector<double> sts(nr);
    for (int r = 0; r < nr; ++r)
      CK(cudaMemcpyAsync(&sts[r], wall + (int64_t)r * (wcap + 1) + wcap, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int worst = 0;
    for (int r = 0; r < nr; ++r) if ((int)sts[r] != 0 && (worst == 0 || (int)sts[r] > worst)) worst = (int)sts[r];
    if (worst) throw MrrrError{worst};
    if (m > 1) { k_monotone<<<1, 1024, 0, s>>>(P.w_all, (int)m); CK(cudaGetLastError()); g_stats.kernel_launches++; }
  };
  h2d(slot_out, h_own.data(), nslots, s);
  *m_out = m;
  if (tr.on) { CK(cudaStreamSynchronize(s)); tr.mark("root bisection"); }
  g_stats.ms_root = tm.stop();
  tl_mark("root done");

  if (!vectors) {
    k_values<<<(nslots + 255) / 256, 256, 0, s>>>(slot_node, slot_out, dnodes, slo, shi,
                                                  (int)nslots, 1.0 / scale, w_loc);
    CK(cudaGetLastError());
    g_stats.kernel_launches++;
    finish_w();
    CK(cudaStreamSynchronize(s));
    g_stats.ms_total = tall.stop();
    g_stats.ms_k_root_bisect = kt_root.ms();
    return 0;
  }
  if (nblocks > 1 && P.m_local > 0)
    CK(cudaMemset2DAsync(P.Z, P.ldz * sizeof(double), 0, n * sizeof(double), P.m_local, s));

  // ---------------- a4/a5: representation tree ----------------
  dump("root_lo.bin", slo, nslots, s);
  dump("root_hi.bin", shi, nslots, s);
  std::vector<int> h_active(nslots, 1);
  int *active = ar.alloc<int>(nslots);
  int *run_end = ar.alloc<int>(nslots);
  std::vector<int> h_run_end(nslots);
  std::vector<VecTask> tasks;
  std::vector<HostNode> hn(nnodes);
  for (int r = 0; r < nroot; ++r) {
    const Block &B = hb[root_blocks[r]];
    hn[B.root_node] = {B.slot0, B.slot1, 0, root_blocks[r]};
  }
  // 1x1 blocks: the vector kernel handles nb == 1 directly
  std::vector<int> level_nodes(h_root_nodes);
  double *wlo = ar.alloc<double>(nslots), *whi = ar.alloc<double>(nslots);
  const int64_t nbmax = [&] { int x = 1; for (auto &B : hb) x = std::max(x, B.nb); return (int64_t)x; }();
  int level = 0;
  unsigned long long h_ctr[48];
  // ---- a6 overlapped with the tree: the singletons a level classifies are
  // final, so their vectors start at once on a lower-priority side stream
  // (events order them after the kernels that produced their node and
  // bracket) while the main stream continues with the next level.
  double *lam = ar.alloc<double>(std::max<int64_t>(nslots, 1));
  int *fail_list = ar.alloc<int>(std::max<int64_t>(nslots, 1)), *fail_count = ar.alloc<int>(1);
  CK(cudaMemsetAsync(fail_count, 0, sizeof(int), s));
  // MRRR_VEC_MODE=1 (diagnostic): all vectors in one batch after the tree
  const int vec_mode = env_int("MRRR_VEC_MODE", 0);
  const int flush_late = env_int("MRRR_FLUSH_LATE", 0);
  const int flush_late_min = env_int("MRRR_FLUSH_LATE_MIN", 64);
  // batches go round-robin to kSide side streams so that they overlap one
  // another as well as the tree (one side stream ran them back to back: the
  // batches are latency-bound, ~12 ms each at n = 20000, and their chain
  // outlasted the tree by ~50 ms)
  // The side streams are created once per host thread and device (creating
  // streams every call cost 10-40 ms per call next to an nvidia-smi sampler);
  // the guard joins them into the call's stream on every exit path.
  struct SideStreams {
    cudaStream_t main, *st;
    ~SideStreams() {
      for (int k = 0; k < kSide; ++k) join_streams_nothrow(main, st[k]);
    }
  } side{s, side_streams()};
  int nbatch = 0;
  // checkpoint columns: one buffer of ck_cap tasks per side stream, reused by
  // the stream's next batch (stream order); a level's singletons go out in
  // pieces of at most ck_cap - 32 tasks, so the checkpoints take
  // kSide * ck_cap * nseg * 48 bytes whatever the batch sizes
  // pieces of (this rank's tasks)/4 (n = 20000: 69.9 -> 67.8 ms against /8),
  // capped so that the checkpoints (64 B per 16-row segment and task) stay
  // within scratch_bytes (16 GB by default; n = 1e5: pieces of ~nslots/10)
  const int nside = std::min(kSide, std::max(1, env_int("MRRR_NSIDE", kNSideDefault)));
  const int piece_div = std::max(1, env_int("MRRR_PIECE_DIV", 4));  // diagnostic knob
  const int64_t ck_mem_cap = (int64_t)(ck_bytes / (64.0 * nside * ((nbmax + kSeg - 1) / kSeg)));
  const int64_t task_basis = dist ? std::min<int64_t>(nslots, wcap + 2) : nslots;
  const int64_t ck_cap =
      std::max<int64_t>(256, std::min<int64_t>((task_basis + piece_div - 1) / piece_div, ck_mem_cap)) + 32;
  const int nseg_v = (int)((nbmax + kSeg - 1) / kSeg);
  FwdCk *ck_f[kSide] = {};
  BwdCk *ck_b[kSide] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> vec_ev;
  std::vector<int> vec_ev_level;  // tree level that launched each piece (MRRR_TIMELINE)
  size_t vec_done = 0;
  // Child RRR slots (nbmax (D+, LLD+) rows each), RECYCLED (SURVEY H9,
  // memory independent of the tree's size).  A node's slot is
  // written by its cluster's child step and read by the refinement of its
  // members (same level), by the child steps of its own clusters (next level:
  // the last reader on the call's stream) and by the vector pieces of its
  // singletons (side streams).  After that child step the slot waits in
  // pool_hold for the pieces holding the node's singletons; it returns to the
  // free list once every one of them has completed (event query, no host
  // wait) and the deferred-fallback counter copied after it reads zero (the
  // fallback re-reads a failed vector's node, reading 10).  So no slot is
  // rewritten before its last reader.  With the vectors after the tree
  // (MRRR_VEC_MODE=1) the slots live until the end, as in round 1.
  std::vector<double2 *> pool_free, node_rrr(nnodes, nullptr);
  std::vector<int> node_pf(nnodes, -1), node_pl(nnodes, -1);  // first / last piece holding a singleton of the node
  struct PoolHold {
    double2 *p;
    int pf, pl;
  };
  std::vector<PoolHold> pool_hold;
  std::vector<cudaEvent_t> piece_done;
  std::vector<volatile int *> piece_fail;  // pinned: the fallback counter after the piece
  std::vector<signed char> piece_ok;      // 1 done, no fallback; 0 done with fallback; -1 running
  int64_t pool_slots = 0;
  // slots for `need` clusters: recycle what is done, then one fresh batch
  auto pool_reserve = [&](int need) {
    for (size_t q = 0; q < piece_done.size(); ++q) {
      if (piece_ok[q] >= 0) continue;
      const cudaError_t st = cudaEventQuery(piece_done[q]);
      if (st == cudaErrorNotReady) continue;
      if (st != cudaSuccess) throw CudaError{st};
      piece_ok[q] = piece_fail[q] != nullptr && *piece_fail[q] == 0 ? 1 : 0;
    }
    size_t k = 0;
    for (size_t h = 0; h < pool_hold.size(); ++h) {
      const PoolHold &H = pool_hold[h];
      bool done = true;
      for (int q = H.pf; q >= 0 && q <= H.pl && done; ++q) done = piece_ok[q] == 1;
      if (done) pool_free.push_back(H.p);
      else pool_hold[k++] = H;
    }
    pool_hold.resize(k);
    const int fresh = need - (int)pool_free.size();
    if (fresh > 0) {
      double2 *b = ar.alloc<double2>((size_t)fresh * nbmax);
      for (int i = fresh - 1; i >= 0; --i) pool_free.push_back(b + (size_t)i * nbmax);
      pool_slots += fresh;
      g_stats.pool_bytes = pool_slots * nbmax * (int64_t)sizeof(double2);
    }
  };
  auto pool_take = [&]() -> double2 * {
    double2 *p = pool_free.back();
    pool_free.pop_back();
    return p;
  };
  auto pool_release_level = [&](const std::vector<int> &nodes_done) {
    if (vec_mode != 0 && vectors) return;
    for (int nd : nodes_done)
      if (nd < (int)node_rrr.size() && node_rrr[nd]) {
        pool_hold.push_back({node_rrr[nd], node_pf[nd], node_pl[nd]});
        node_rrr[nd] = nullptr;
      }
  };
  // streamed download (host entry, pinned Z): a block of kZB columns goes to
  // the host on the copy stream once every piece that writes into it has been
  // launched, after those pieces' events -- the D2H of Z (3.2 GB at n = 20000)
  // overlaps the rest of the solve instead of following it
  // (measured, n = 20000: 32 / 64 / 256 / 1024 columns per block -> e2e 101.7 /
  // 102.1 / 105.3 / 102.9 ms; copying each piece's own column runs instead --
  // 810-2485 copies -- 107.8-134.6 ms: the columns of a level's singletons are
  // only ready when its piece ends, late in the solve, and the small copies
  // cost more than they overlap.  MRRR_ZB: diagnostic)
  const int64_t kZB = std::max(1, env_int("MRRR_ZB", 64));
  const bool zstream = P.hZ != nullptr && vectors && P.m_local > 0;
  cudaStream_t sc = zstream ? copy_stream() : nullptr;
  // the copy stream rejoins the solve stream on EVERY exit (an error after
  // some Z blocks were queued must not let the host entry free dZ, or the
  // caller its host buffer, while a download still runs)
  struct CopyJoin {
    cudaStream_t main, sc;
    ~CopyJoin() { join_streams_nothrow(main, sc); }
  } cjoin{s, sc};
  const int64_t nzb = zstream ? (P.m_local + kZB - 1) / kZB : 0;
  std::vector<int64_t> zb_left(nzb, 0);
  std::vector<std::vector<cudaEvent_t>> zb_ev(nzb);
  if (zstream) {
    for (int q = 0; q < (int)nslots; ++q)
      if (h_own[q] >= 0) ++zb_left[h_own[q] / kZB];
    cudaEvent_t e0 = ev_sync();  // Z's memset (split matrices) precedes every copy
    CK(cudaEventRecord(e0, s));
    CK(cudaStreamWaitEvent(sc, e0, 0));
  }
  auto zb_copy = [&](int64_t c0, int64_t c1) {  // columns [c0, c1) after sc's pending waits
    CK(cudaMemcpy2DAsync(P.hZ + c0 * P.hldz, P.hldz * sizeof(double), P.Z + c0 * P.ldz,
                         P.ldz * sizeof(double), n * sizeof(double), c1 - c0, cudaMemcpyDeviceToHost, sc));
    ++g_stats.z_copies;
  };
  auto zb_done = [&](size_t t0, size_t t1, cudaEvent_t eb) {  // tasks [t0, t1) written after eb
    if (!zstream) return;
    for (size_t t = t0; t < t1; ++t) {
      const int64_t b = tasks[t].col / kZB;
      if (zb_ev[b].empty() || zb_ev[b].back() != eb) zb_ev[b].push_back(eb);
      if (--zb_left[b] == 0) {
        for (cudaEvent_t e : zb_ev[b]) CK(cudaStreamWaitEvent(sc, e, 0));
        zb_copy(b * kZB, std::min<int64_t>(P.m_local, (b + 1) * kZB));
      }
    }
  };
  // pieces that overlap a heavy tree level run on single warps (smaller
  // footprint next to the tree's kernels); the last flush, and pieces whose
  // level leaves at most kPairWork cluster-rows (clusters x block order) to
  // step and refine, on warp pairs (half the latency).  Measured (B200):
  // random n=20000 (<= 1049 clusters x 2e4 rows per level) 53.6 -> 51.3 ms
  // with pairs at every level, glued n=21000 71.0 -> 69.6 ms, but random
  // n=1e5 (221-1173 clusters x 1e5 rows) 1084 -> 1133 ms: there the longer
  // pair pieces crowd the tree's kernels.  MRRR_VEC_PAIR: 0 never, 2 always;
  // MRRR_PAIR_WORK overrides the bound (diagnostic).
  const double kPairWork = getenv("MRRR_PAIR_WORK") ? atof(getenv("MRRR_PAIR_WORK")) : 2.5e7;
  const int vec_pair = env_int("MRRR_VEC_PAIR", 1);
  const int vec_split = env_int("MRRR_VEC_SPLIT", 1);
  // warp-pair pieces with the lanes regrouped by twist index too
  // (k_wvectors_psplit); MRRR_VEC_PSPLIT=0: k_wvectors_pair (diagnostic)
  const int vec_psplit = env_int("MRRR_VEC_PSPLIT", 1);
  const int vec_pack = env_int("MRRR_VEC_PACK", 1) ? kMaxSeg : 1;
  const int tree_side = std::min(nside, std::max(1, env_int("MRRR_TREE_SIDE", nside)));
  // Which side stream takes the next piece: the first idle one in
  // round-robin order (its last piece's end event has completed), else the
  // one whose last piece was launched first.  Together with pieces of equal
  // size per flush (below) this keeps a flush's pieces off each other's
  // streams and puts them behind the pieces that started earliest.  Measured
  // (random n = 20000, profiles/r02/setE): round robin with a full-size +
  // remainder split 35.6 ms (a level-3 piece queued behind the longest
  // level-2 piece, 6.8 ms vector tail); equal pieces 33.9 ms; the stream
  // with the fewest queued tasks 37.1 ms (it put the two pieces of one flush
  // on one stream).  The choice only moves pieces between streams: results
  // are the same on any stream (test_schedule_invariance).
  int side_last[kSide];
  for (int k = 0; k < kSide; ++k) side_last[k] = -1;
  auto pick_side = [&](int ns) {
    if (env_int("MRRR_SIDE_RR", 0)) return nbatch % ns;  // diagnostic: round robin
    for (int q = 0; q < ns; ++q) {
      const int k = (nbatch + q) % ns;
      if (side_last[k] < 0) return k;
      const cudaError_t st = cudaEventQuery(piece_done[side_last[k]]);
      if (st == cudaSuccess) return k;
      if (st != cudaErrorNotReady) throw CudaError{st};
    }
    int best = 0;
    for (int k = 1; k < ns; ++k)
      if (side_last[k] < side_last[best]) best = k;
    return best;
  };
  auto flush_vectors = [&](int tree_left) {
    // a flush's tasks in pieces of equal size (<= ck_cap - 32 each): with
    // full pieces plus a remainder the remainder piece ended ~4 ms before
    // the full ones it was launched with
    const size_t nflush = tasks.size() - vec_done, pmax = (size_t)(ck_cap - 32);
    const size_t npiece = (nflush + pmax - 1) / pmax;
    const size_t pchunk = npiece > 0 ? (nflush + npiece - 1) / npiece : pmax;
    for (size_t t0 = vec_done; t0 < tasks.size();) {
      const size_t t1 = std::min<size_t>(tasks.size(), t0 + pchunk);
      const int nbt = (int)(t1 - t0);
      std::vector<VecTask> bt(tasks.begin() + t0, tasks.begin() + t1);
      VecTask *dtb = ar.alloc<VecTask>(nbt);
      // side streams: tree_side of them while the tree runs (fewer vector
      // warps next to its kernels), all kSide for the last flush
      const int sk = pick_side(tree_left > 0 ? tree_side : nside);
      if (!ck_f[sk]) {
        ck_f[sk] = ar.alloc<FwdCk>((size_t)nseg_v * ck_cap);
        ck_b[sk] = ar.alloc<BwdCk>((size_t)nseg_v * ck_cap);
      }
      auto items = make_warp_items(bt, hn, vec_pack);
      g_stats.vec_items += (int64_t)items.size();
      WarpItem *ditems = ar.alloc<WarpItem>(items.size());
      h2d(dtb, bt.data(), nbt, s);
      h2d(ditems, items.data(), items.size(), s);
      cudaEvent_t ready = ev_sync();
      CK(cudaEventRecord(ready, s));
      cudaStream_t s2 = side.st[sk];
      ++nbatch;
      CK(cudaStreamWaitEvent(s2, ready, 0));
      WVecArgs A{};
      A.nodes = dnodes; A.LDv = LDv; A.tasks = dtb; A.items = ditems; A.nitems = (int)items.size();
      A.lo = slo; A.hi = shi; A.fck = ck_f[sk]; A.bck = ck_b[sk]; A.ck_stride = ck_cap; A.ntask = nbt;
      A.Z = P.Z; A.ldz = P.ldz; A.lam_out = lam + t0; A.mode = 0; A.ctr = ctr + 8; A.hist = ctr + 32;
      A.slot_j = slot_j; A.rqc_max = std::max(1, P.o.rqc_max);
      A.fail_list = fail_list; A.fail_count = fail_count; A.task_base = (int)t0;
      const bool pair = vec_pair == 2 || (vec_pair == 1 && (double)tree_left * (double)nbmax <= kPairWork);
      // single-warp pieces: split RQC with the lanes regrouped by twist index
      // between the phases (k_wvectors_split: ~25 % fewer rows walked by the
      // fixed-twist factorizations and the solve; random n = 1e5 1.84 -> 1.59 s).
      // MRRR_VEC_SPLIT=0: one kernel (k_wvectors).
      const bool split = vec_split != 0 && (!pair || vec_psplit != 0);
      SplitBufs sb{};
      if (split) {
        // sort segments: each node's run of tasks (items may span several nodes)
        std::vector<int> seg_b, seg_e;
        for (int q = 0; q < nbt; ++q)
          if (q == 0 || bt[q].node != bt[q - 1].node) { seg_b.push_back(q); seg_e.push_back(q + 1); }
          else seg_e.back() = q + 1;
        sb.nseg = (int)seg_b.size();
        sb.state = ar.alloc<RqcState>(nbt);
        sb.rkey = ar.alloc<int>(nbt); sb.rkey_out = ar.alloc<int>(nbt);
        sb.perm_in = ar.alloc<int>(nbt); sb.perm = ar.alloc<int>(nbt);
        sb.seg_b = ar.alloc<int>(sb.nseg); sb.seg_e = ar.alloc<int>(sb.nseg);
        h2d(sb.seg_b, seg_b.data(), sb.nseg, s);
        h2d(sb.seg_e, seg_e.data(), sb.nseg, s);
        sb.bits = 1;
        while ((int64_t(1) << sb.bits) < nbmax) ++sb.bits;
        CK(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, sb.temp_bytes, sb.rkey, sb.rkey_out, sb.perm_in,
                                                    sb.perm, nbt, sb.nseg, sb.seg_b, sb.seg_e, 0, sb.bits, s2));
        sb.temp = ar.alloc<char>(sb.temp_bytes);
        // (the uploads above are on the call's stream: record `ready` after them)
        cudaEvent_t ready2 = ev_sync();
        CK(cudaEventRecord(ready2, s));
        CK(cudaStreamWaitEvent(s2, ready2, 0));
      }
      NvtxScope nvtx_piece("mrrr vector piece");
      cudaEvent_t ea = ev_time(), eb = ev_time();
      CK(cudaEventRecord(ea, s2));
      if (split) {
        A.state = sb.state; A.rkey = sb.rkey;
        if (pair) launch_wpsplit(A, 3, s2);
        else launch_wsplit(A, 3, s2);
        k_iota<<<(nbt + 255) / 256, 256, 0, s2>>>(sb.perm_in, nbt);
        CK(cub::DeviceSegmentedRadixSort::SortPairs(sb.temp, sb.temp_bytes, sb.rkey, sb.rkey_out, sb.perm_in,
                                                    sb.perm, nbt, sb.nseg, sb.seg_b, sb.seg_e, 0, sb.bits, s2));
        A.task_list = sb.perm;
        if (pair) launch_wpsplit(A, 4, s2);
        else launch_wsplit(A, 4, s2);
        g_stats.kernel_launches += 2;
      } else {
        launch_wvec(A, s2, pair);
      }
      {
        // the deferred-fallback counter after this piece (pool_collect)
        volatile int *pfc = (volatile int *)g_staging.get(sizeof(int));
        if (pfc) {
          *pfc = -1;
          CK(cudaMemcpyAsync((void *)pfc, fail_count, sizeof(int), cudaMemcpyDeviceToHost, s2));
        }
        const int pc = (int)piece_done.size();
        side_last[sk] = pc;
        piece_done.push_back(eb);
        piece_fail.push_back(pfc);
        piece_ok.push_back(-1);
        for (const VecTask &t : bt) {
          if (t.node >= (int)node_pf.size()) continue;
          if (node_pf[t.node] < 0) node_pf[t.node] = pc;
          node_pl[t.node] = pc;
        }
      }
      CK(cudaEventRecord(eb, s2));
      tr.fine(s2, "  vectors (side stream)");
      vec_ev.push_back({ea, eb});
      vec_ev_level.push_back(tl_level);
      zb_done(t0, t1, eb);
      t0 = t1;
    }
    vec_done = tasks.size();
  };
  Timer ttree(s);
  for (;;) {
    {
      char nm[32];
      snprintf(nm, sizeof nm, "mrrr level %d", level);
      tr.phase(nm);
    }
    tl_level = level;
    tl_mark("L" + std::to_string(level) + " start");
    h2d(active, h_active.data(), nslots, s);
    k_classify<<<(nslots + 255) / 256, 256, 0, s>>>(slot_node, slo, shi, active, (int)nslots,
                                                    P.o.tol_relgap, run_end);
    CK(cudaGetLastError());
    g_stats.kernel_launches++;
    d2h(h_run_end.data(), run_end, nslots, s);
    tr.mark("classify");
    if (level == 0 && dist && nblocks == 1 && m > 1) {
      // e: the shard planner -- every cut moves to the nearest root-cluster
      // boundary within epp / 40 (identical on every rank: the root brackets
      // were exchanged), before any vector is assigned
      std::vector<unsigned char> free_cut(m + 1, 0);
      for (int64_t j = 1; j < m; ++j) free_cut[j] = h_run_end[col_slot[j - 1]] != 0;
      plan_columns(m, nr, free_cut.data(), cuts.data());
      apply_cuts();
    }
    // the level's clusters: identical on every rank (the brackets are
    // exchanged after each refinement); a rank works on the clusters that
    // hold one of its columns ("own")
    std::vector<int> cl_parent, cl_s0, cl_s1, own_cl;
    for (int nd : level_nodes) {
      const HostNode &H = hn[nd];
      int st = H.slot0;
      for (int q = H.slot0; q < H.slot1; ++q) {
        if (!h_active[q]) { st = q + 1; continue; }
        if (h_run_end[q]) {
          if (q == st) {
            if (h_own[q] >= 0) {
              VecTask t; t.slot = q; t.node = nd; t.col = h_own[q]; t.lam0 = NAN;
              tasks.push_back(t);
            }
            h_active[q] = 0;
          } else {
            bool wanted = false, own = false;
            for (int x = st; x <= q; ++x) { wanted |= h_slot_out[x] >= 0; own |= h_own[x] >= 0; }
            if (wanted) {
              if (own) own_cl.push_back((int)cl_parent.size());
              cl_parent.push_back(nd); cl_s0.push_back(st); cl_s1.push_back(q + 1);
            } else {
              for (int x = st; x <= q; ++x) h_active[x] = 0;
            }
          }
          st = q + 1;
        }
      }
    }
    const int ncl = (int)cl_parent.size(), nown = (int)own_cl.size();
    // When the level's singletons go out: at the level's start, or (flush_late,
    // levels with at least flush_late_min clusters) behind the level's cluster
    // step, so that the step's kernels do not share the SMs' registers with
    // the new pieces (see the note at the late flush below)
    const bool late_flush = vectors && vec_mode == 0 && flush_late && ncl >= flush_late_min;
    if (vectors && (vec_mode == 0 || ncl == 0) && !late_flush) guarded([&] { flush_vectors(nown); });
    if (ncl == 0) break;
    if (level + 1 > P.o.max_depth) throw MrrrError{MRRR_ERR_DEPTH};  // the same level on every rank
    g_stats.nodes += nown;
    // grow node table
    int node_base = nnodes;
    guarded([&] {
    if (nnodes + ncl > node_cap) {
      int ncap = std::max(node_cap * 2, nnodes + ncl + 16);
      Node *nn = ar.alloc<Node>(ncap);
      CK(cudaMemcpyAsync(nn, dnodes, nnodes * sizeof(Node), cudaMemcpyDeviceToDevice, s));
      dnodes = nn; node_cap = ncap;
    }
    // per-level scratch, released (to the library pool) at the end of the level
    DevArena lv(device_ws(g_ws_level));
    std::vector<int> ocl_parent(nown), ocl_s0(nown), ocl_s1(nown);
    for (int i = 0; i < nown; ++i) {
      const int c = own_cl[i];
      ocl_parent[i] = cl_parent[c]; ocl_s0[i] = cl_s0[c]; ocl_s1[i] = cl_s1[c];
    }
    int *dcl_parent = lv.alloc<int>(ncl), *dcl_s0 = lv.alloc<int>(ncl), *dcl_s1 = lv.alloc<int>(ncl);
    int *docl_parent = lv.alloc<int>(nown + 1), *docl_s0 = lv.alloc<int>(nown + 1), *docl_s1 = lv.alloc<int>(nown + 1);
    int *down_cl = lv.alloc<int>(nown + 1);
    h2d(dcl_parent, cl_parent.data(), ncl, s);
    h2d(dcl_s0, cl_s0.data(), ncl, s);
    h2d(dcl_s1, cl_s1.data(), ncl, s);
    h2d(docl_parent, ocl_parent.data(), nown, s);
    h2d(docl_s0, ocl_s0.data(), nown, s);
    h2d(docl_s1, ocl_s1.data(), nown, s);
    h2d(down_cl, own_cl.data(), nown, s);
    // a5 cluster step on the own clusters: probes, six candidates, choice,
    // chosen child (one kernel).  The step's scratch (kCSRows rows of nbmax
    // doubles per cluster) is capped at 16 GB: beyond, clusters go through in
    // groups that reuse it (stream order; each group costs one more chain latency)
    int cgrp = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(nown, 1), (int64_t)(scratch_bytes / (8.0 * kCSRows * nbmax))));
    if (env_int("MRRR_CS_GROUP", 0) > 0) cgrp = std::min(cgrp, env_int("MRRR_CS_GROUP", 0));  // test hook
    const int64_t zs_cs = (nbmax + 7) / 8 * 8;  // scratch row stride (q every 8 rows needs ceil(nb / 8) per candidate)
    double *scratch = nown ? (double *)grow_buffer(child_scratch(), (size_t)kCSRows * cgrp * zs_cs * sizeof(double)) : nullptr;
    if (nown) cs_scratch_used = std::max(cs_scratch_used, (size_t)kCSRows * cgrp * zs_cs * sizeof(double));
    double *dsig_own = lv.alloc<double>(nown + 1), *dsig = lv.alloc<double>(ncl);
    int *dtier = lv.alloc<int>(nown + 1);
    // child RRR slots of the own clusters (recycled: pool_take)
    std::vector<double2 *> cl_rrr(ncl, nullptr), own_rrr(std::max(nown, 1), nullptr);
    pool_reserve(nown);
    for (int i = 0; i < nown; ++i) own_rrr[i] = cl_rrr[own_cl[i]] = pool_take();
    double2 **dcl_rrr = lv.alloc<double2 *>(ncl), **down_rrr = lv.alloc<double2 *>(std::max(nown, 1));
    h2d(dcl_rrr, cl_rrr.data(), ncl, s);
    h2d(down_rrr, own_rrr.data(), nown, s);
    node_rrr.resize(node_base + ncl, nullptr);
    node_pf.resize(node_base + ncl, -1);
    node_pl.resize(node_base + ncl, -1);
    for (int c = 0; c < ncl; ++c) node_rrr[node_base + c] = cl_rrr[c];
    tr.fine(s, "  alloc+upload");
    if (tr.lvl >= 2) {
      unsigned z[64] = {};
      CK(cudaMemcpyToSymbol(g_rw_hist, z, sizeof z));
    }
    int h_fail[4] = {0, 0, 0, 0};
    {
      // clusters of >= 2000 members (reading 30) go through the nine-warp
      // step with the interior candidate, in their own launch and scratch;
      // the others through the five-warp step, in groups that fit the scratch
      const bool child_v1 = child_v1_env >= 0 ? child_v1_env != 0 : nown <= kChildV1Max;
      const bool child_v3 = !child_v1 && child_v3_env != 0;
      cudaStream_t big_stream = nullptr;
      struct BigJoin {  // the second stream rejoins the solve stream on every exit
        cudaStream_t main, b;
        ~BigJoin() { if (b) join_streams_nothrow(main, b); }
      } bjoin{s, nullptr};
      std::vector<int> small_cl, big_cl;
      for (int i = 0; i < nown; ++i)
        (P.o.shift_strategy == 1 && ocl_s1[i] - ocl_s0[i] >= 2000 ? big_cl : small_cl).push_back(i);
      auto child_args = [&](const int *list, int c0, int c1, double *scr) {
        ChildArgs C{};
        C.nodes = dnodes; C.cl_parent = docl_parent; C.cl_s0 = docl_s0; C.cl_s1 = docl_s1;
        C.lo = slo; C.hi = shi; C.LDv = LDv; C.c0 = c0; C.ncl = c1;
        C.rtol = P.o.rtol_class;
        C.scratch = scr; C.zstride = zs_cs;
        C.pool = down_rrr; C.sigma_out = dsig_own; C.tier_out = dtier; C.fail = dfail + 1;
        C.ctr = ctr + 16;
        C.shift_strategy = P.o.shift_strategy;
        C.int_wg = int_wg;
        C.cl_list = list;
        return C;
      };
      if (!big_cl.empty()) {
        const int nbig = (int)big_cl.size();
        int *dbig = lv.alloc<int>(nbig);
        h2d(dbig, big_cl.data(), nbig, s);
        double *scr = lv.alloc<double>((size_t)kCSRowsAdj * nbig * zs_cs);
        // on a second high-priority stream, beside the other clusters' step
        // (forked after the uploads above, joined before k_child_nodes)
        big_stream = hp_stream2();
        bjoin.b = big_stream;
        cudaEvent_t fork = ev_sync();
        CK(cudaEventRecord(fork, s));
        CK(cudaStreamWaitEvent(big_stream, fork, 0));
        if (child_v1) k_child_step<1><<<nbig, 32 * kCSWarpsAdj, 0, big_stream>>>(child_args(dbig, 0, nbig, scr));
        else k_child_step2<1><<<nbig, 96, 0, big_stream>>>(child_args(dbig, 0, nbig, scr));
        CK(cudaGetLastError());
        g_stats.kernel_launches++;
      }
      const int nsmall = (int)small_cl.size();
      int *dsmall = nullptr;
      if (!big_cl.empty() && nsmall) {
        dsmall = lv.alloc<int>(nsmall);
        h2d(dsmall, small_cl.data(), nsmall, s);
      }
      for (int c0 = 0; c0 < nsmall; c0 += cgrp) {
        const int nl = std::min(nsmall, c0 + cgrp) - c0;
        if (child_v1) {
          k_child_step<0><<<nl, 32 * kCSWarps, 0, s>>>(child_args(dsmall, c0, c0 + nl, scratch));
        } else if (child_v3) {
          // chains lane-dense (three clusters per warp), then the rest of the step
          const int per = c3_groups * kC3Warps;
          const ChildArgs CA = child_args(dsmall, c0, c0 + nl, scratch);
          if (c3_groups == 1) k_child_chains3<1><<<(nl + per - 1) / per, 32 * kC3Warps, 0, s>>>(CA);
          else if (c3_groups == 2) k_child_chains3<2><<<(nl + per - 1) / per, 32 * kC3Warps, 0, s>>>(CA);
          else k_child_chains3<3><<<(nl + per - 1) / per, 32 * kC3Warps, 0, s>>>(CA);
          CK(cudaGetLastError());
          k_child_step2<0, true><<<nl, 128, 0, s>>>(child_args(dsmall, c0, c0 + nl, scratch));
          g_stats.kernel_launches++;
        } else {
          k_child_step2<0><<<nl, 96, 0, s>>>(child_args(dsmall, c0, c0 + nl, scratch));
        }
        CK(cudaGetLastError());
        g_stats.kernel_launches++;
      }
      if (big_stream) {  // join the big clusters' step
        cudaEvent_t join = ev_sync();
        CK(cudaEventRecord(join, big_stream));
        CK(cudaStreamWaitEvent(s, join, 0));
        bjoin.b = nullptr;
      }
      tr.fine(s, "  child step");
      tl_mark("L" + std::to_string(level) + " child step done");
      if (tr.lvl >= 2) {  // diagnostic: this level's slowest cluster step, cycles per phase
        unsigned long long c[8];
        CK(cudaMemcpy(c, ctr + 16, sizeof c, cudaMemcpyDeviceToHost));
        fprintf(stderr, "[mrrr]   child step cycles (%s): candidates %llu, probe bwd %llu, probe fwd %llu; "
                "twist+scan %llu; growth %llu\n", child_v1 ? "v1" : "v2", c[2], c[3], c[4], c[5], c[6]);
        const unsigned long long z[5] = {0, 0, 0, 0, 0};
        CK(cudaMemcpy(ctr + 18, z, sizeof z, cudaMemcpyHostToDevice));
        std::vector<int> ht(std::max(nown, 1));
        CK(cudaMemcpy(ht.data(), dtier, nown * sizeof(int), cudaMemcpyDeviceToHost));
        int tc[8] = {};
        for (int i = 0; i < nown; ++i) tc[std::min(std::max(ht[i], 0), 7)]++;
        fprintf(stderr, "[mrrr]   child tiers: (i) %d, (ii) %d, (iii) %d, none %d, interior %d\n", tc[0], tc[1],
                tc[3], tc[4], tc[5]);
      }
      g_stats.child_sweeps += 7 * nown;
      // sigma of every cluster of the level (0 where another rank owns it:
      // those members' brackets arrive by the exchange below)
      CK(cudaMemsetAsync(dsig, 0, ncl * sizeof(double), s));
      if (nown) k_scatter<<<(nown + 255) / 256, 256, 0, s>>>(down_cl, dsig_own, nown, dsig);
      // the child node entries are written before the translate kernel reads sigma
      k_child_nodes<<<(ncl + 63) / 64, 64, 0, s>>>(dnodes, node_base, dcl_parent, dcl_s0, dcl_s1, dsig, ncl,
                                                   dcl_rrr, slot_j);
      // late flush: the pieces wait for the cluster step (event on this stream)
      // and are registered with their nodes before the parents' slots are released
      if (late_flush) flush_vectors(nown);
      // the parents' RRRs (read by the child step above, last reader on this
      // stream) go back to the pool once their vector pieces are done
      pool_release_level(level_nodes);
      CK(cudaGetLastError());
      // translate member brackets to child coordinates
      std::vector<int> slot_cl, first_slot;
      for (int c = 0; c < ncl; ++c)
        for (int q = cl_s0[c]; q < cl_s1[c]; ++q) { slot_cl.push_back(c); first_slot.push_back(q); }
      int nsn = (int)slot_cl.size();
      int *dslot_cl = lv.alloc<int>(nsn), *dfirst = lv.alloc<int>(nsn);
      h2d(dslot_cl, slot_cl.data(), nsn, s);
      h2d(dfirst, first_slot.data(), nsn, s);
      k_translate<<<(nsn + 127) / 128, 128, 0, s>>>(dslot_cl, dfirst, nsn, dsig, slo, shi, wlo, whi,
                                                    slot_node, node_base);
      CK(cudaGetLastError());
      g_stats.kernel_launches += 3;
      // verify + refine in child coordinates: chunks of rw_chunk_tree(m)
      // members from each cluster's start -- the refinement of a chunk depends
      // on the chunk alone, so ranks sharing a cluster compute bitwise the same
      // brackets; a rank refines the chunks holding one of its slots (§8(e),
      // the paper's type-3 task)
      std::vector<Work> wv, all;
      for (int i = 0; i < nown; ++i) {
        const int c = own_cl[i];
        all.clear();
        const int mcl = cl_s1[c] - cl_s0[c];
        if (rw_end > 0 && mcl >= rw_end) {
          // the two end members alone (the child's shift sits next to one of
          // them: in child coordinates it needs ~20 more bits than the rest,
          // and alone its warp gives it all 32 shifts from the first round)
          make_work(node_base + c, cl_s0[c], cl_s0[c] + 1, 1, all);
          make_work(node_base + c, cl_s0[c] + 1, cl_s1[c] - 1, rw_chunk_tree(mcl), all);
          make_work(node_base + c, cl_s1[c] - 1, cl_s1[c], 1, all);
        } else {
          make_work(node_base + c, cl_s0[c], cl_s1[c], rw_chunk_tree(mcl), all);
        }
        for (const Work &W : all) {
          bool mine = !dist;
          for (int q = W.s0; q < W.s1 && !mine; ++q) mine = h_slot_owner[q] == P.rank;
          if (mine) wv.push_back(W);
        }
      }
      Work *dwork = lv.alloc<Work>(wv.size() + 1);
      h2d(dwork, wv.data(), wv.size(), s);
      launch_refine(dnodes, dwork, (int)wv.size(), nullptr, slot_j, slo, shi, wlo, whi, 1, P.o.rtol_class,
                    dfail + 2, ctr + 2, ctr + 1, s, rw_m_tree, early_bits > 0 ? P.o.tol_relgap : 0.0,
                    std::ldexp(1.0, -early_bits), split_tree);
      tr.fine(s, "  refine");
      tl_mark("L" + std::to_string(level) + " refine done");
      if (tr.lvl >= 2) {  // diagnostic: rounds per refinement warp
        unsigned hist[64];
        CK(cudaMemcpyFromSymbol(hist, g_rw_hist, sizeof hist));
        fprintf(stderr, "[mrrr]   refine rounds histogram:");
        for (int r = 0; r < 64; ++r)
          if (hist[r]) fprintf(stderr, " %d:%u", r, hist[r]);
        fprintf(stderr, "\n");
        memset(hist, 0, sizeof hist);
        CK(cudaMemcpyToSymbol(g_rw_hist, hist, sizeof hist));
      }
      d2h(h_fail, dfail, 4, s);
      tl_mark("L" + std::to_string(level) + " flags read");
      if (getenv("MRRR_DUMP")) {
        char nm[64];
        {
          double2 *pc = lv.alloc<double2>((size_t)std::max(nown, 1) * nbmax);
          for (int i = 0; i < nown; ++i)
            CK(cudaMemcpyAsync(pc + (size_t)i * nbmax, own_rrr[i], nbmax * sizeof(double2), cudaMemcpyDeviceToDevice, s));
          snprintf(nm, sizeof nm, "L%d_pool.bin", level); dump(nm, pc, (size_t)nown * nbmax, s);
        }
        snprintf(nm, sizeof nm, "L%d_sigma.bin", level); dump(nm, dsig, ncl, s);
        snprintf(nm, sizeof nm, "L%d_tier.bin", level); dump(nm, dtier, nown, s);
        snprintf(nm, sizeof nm, "L%d_s0.bin", level); dump(nm, dcl_s0, ncl, s);
        snprintf(nm, sizeof nm, "L%d_s1.bin", level); dump(nm, dcl_s1, ncl, s);
        snprintf(nm, sizeof nm, "L%d_parent.bin", level); dump(nm, dcl_parent, ncl, s);
        snprintf(nm, sizeof nm, "L%d_lo.bin", level); dump(nm, slo, nslots, s);
        snprintf(nm, sizeof nm, "L%d_hi.bin", level); dump(nm, shi, nslots, s);
      }
      if (h_fail[1]) throw MrrrError{MRRR_ERR_CHILD};
      if (h_fail[2]) throw MrrrError{MRRR_ERR_CONVERGE};
      if (dist && env_int("MRRR_TEST_FAIL_RANK", -1) == P.rank && level == env_int("MRRR_TEST_FAIL_LEVEL", 0))
        throw MrrrError{MRRR_ERR_CHILD};  // test hook: one rank fails alone (tests/test_gpu_dist.py)
    }
    });  // guarded: reported at the exchange below, where every rank stops
    // e: the level's exchange -- every rank gets the brackets of all members
    // (and the check that all ranks agree on the tree: the global cluster
    // count); an error on any rank stops all ranks here
    if (dist) {
      const double mx = exchange_brackets((double)ncl);
      if ((int)mx != ncl) throw MrrrError{MRRR_ERR_COMM};
    }
    // host mirror (every rank keeps the whole tree's structure: the next
    // level's clusters are classified from the exchanged brackets, so all
    // ranks list the same clusters and run the same number of levels)
    hn.resize(nnodes + ncl);
    for (int c = 0; c < ncl; ++c) {
      hn[node_base + c] = {cl_s0[c], cl_s1[c], hn[cl_parent[c]].depth + 1, hn[cl_parent[c]].block};
      for (int q = cl_s0[c]; q < cl_s1[c]; ++q) h_slot_node[q] = node_base + c;
    }
    nnodes += ncl;
    if (tr.on) {
      char buf[96];
      snprintf(buf, sizeof buf, "level %d: %d clusters (%d here)", level, ncl, nown);
      tr.mark(buf);
    }
    level_nodes.clear();
    for (int c = 0; c < ncl; ++c) level_nodes.push_back(node_base + c);
    ++level;
  }
  g_stats.levels = level;
  g_stats.ms_tree = ttree.stop();
  tl_mark("tree done");

  // ---------------- a6: singleton vectors (launched per level above) ----------------
  tr.phase("mrrr vector tail");
  Timer tv(s);
  const int ntask = (int)tasks.size();
  g_stats.singletons = ntask;
  {
    // join the side streams
    for (int k = 0; k < kSide; ++k) {
      cudaStream_t x = side.st[k];
      cudaEvent_t j = ev_sync();
      CK(cudaEventRecord(j, x));
      CK(cudaStreamWaitEvent(s, j, 0));
    }
  }
  guarded([&] {
  if (ntask > 0) {
    VecTask *dt = ar.alloc<VecTask>(ntask);
    h2d(dt, tasks.data(), ntask, s);
    {
      std::vector<Node> hnodes(nnodes);
      d2h(hnodes.data(), dnodes, nnodes, s);
      int64_t el = 0;
      for (auto &t : tasks) el += hnodes[t.node].nb;
      g_stats.vec_tasks = ntask;
      g_stats.vec_elems = el;
    }
    // deferred O10 fallback (reading 10): brackets of the tasks whose RQC did
    // not converge are refined to 4 eps, then one factorization at the
    // midpoint writes their vectors (mode 2)
    {
      int h_nf = 0;
      d2h(&h_nf, fail_count, 1, s);
      if (h_nf > 0) {
        std::vector<int> fl(h_nf);
        d2h(fl.data(), fail_list, h_nf, s);
        std::sort(fl.begin(), fl.end(), [&](int a, int b) {
          return tasks[a].node != tasks[b].node ? tasks[a].node < tasks[b].node : a < b;
        });
        std::vector<int> slots(h_nf);
        std::vector<VecTask> ft(h_nf);
        std::vector<Work> wv;
        for (int q0 = 0; q0 < h_nf;) {
          int q1 = q0;
          while (q1 < h_nf && tasks[fl[q1]].node == tasks[fl[q0]].node) ++q1;
          for (int a = q0; a < q1; a += 8) {
            Work W; W.node = tasks[fl[q0]].node; W.s0 = a; W.s1 = std::min(a + 8, q1); W.pad = 0;
            wv.push_back(W);
          }
          q0 = q1;
        }
        for (int q = 0; q < h_nf; ++q) { slots[q] = tasks[fl[q]].slot; ft[q] = tasks[fl[q]]; }
        auto fitems = make_warp_items(ft, hn, vec_pack);
        int *dslots = ar.alloc<int>(h_nf), *dfl = ar.alloc<int>(h_nf);
        h2d(dslots, slots.data(), h_nf, s);
        h2d(dfl, fl.data(), h_nf, s);
        Work *dw = ar.alloc<Work>(wv.size());
        h2d(dw, wv.data(), wv.size(), s);
        kt_fin.start(s);
        launch_refine(dnodes, dw, (int)wv.size(), dslots, slot_j, slo, shi, nullptr, nullptr, 0, 4.0 * kEps,
                      dfail + 2, ctr + 2, ctr + 1, s);
        kt_fin.stop(s);
        {
          int hf[4];
          d2h(hf, dfail, 4, s);
          if (hf[2]) throw MrrrError{MRRR_ERR_CONVERGE};  // the fallback's bisection did not converge
        }
        VecTask *dft = ar.alloc<VecTask>(h_nf);
        h2d(dft, ft.data(), h_nf, s);
        WarpItem *dfi = ar.alloc<WarpItem>(fitems.size());
        h2d(dfi, fitems.data(), fitems.size(), s);
        double *lam_c = ar.alloc<double>(h_nf);
        WVecArgs F{};
        F.nodes = dnodes; F.LDv = LDv; F.tasks = dft; F.items = dfi; F.nitems = (int)fitems.size();
        F.lo = slo; F.hi = shi; F.slot_j = slot_j; F.ntask = h_nf; F.ck_stride = h_nf + 32;
        F.fck = ar.alloc<FwdCk>((size_t)nseg_v * (h_nf + 32));
        F.bck = ar.alloc<BwdCk>((size_t)nseg_v * (h_nf + 32));
        F.Z = P.Z; F.ldz = P.ldz; F.lam_out = lam_c; F.mode = 2; F.ctr = ctr + 8;
        launch_wvec(F, s, vec_pair != 0);
        k_scatter<<<(h_nf + 255) / 256, 256, 0, s>>>(dfl, lam_c, h_nf, lam);
        CK(cudaGetLastError());
        g_stats.kernel_launches++;
        if (zstream) {  // the fallback rewrote these columns: download them again
          cudaEvent_t ef = ev_sync();
          CK(cudaEventRecord(ef, s));
          CK(cudaStreamWaitEvent(sc, ef, 0));
          for (int q = 0; q < h_nf; ++q) zb_copy(tasks[fl[q]].col, tasks[fl[q]].col + 1);
        }
      }
    }
    if (zstream) {
      // blocks with columns no piece wrote (none expected): download after all work
      cudaEvent_t ez = ev_sync();
      CK(cudaEventRecord(ez, s));
      for (int64_t b = 0; b < nzb; ++b)
        if (zb_left[b] > 0) {
          CK(cudaStreamWaitEvent(sc, ez, 0));
          zb_copy(b * kZB, std::min<int64_t>(P.m_local, (b + 1) * kZB));
        }
      cudaEvent_t ej = ev_sync();  // the call's stream waits for the downloads
      CK(cudaEventRecord(ej, sc));
      CK(cudaStreamWaitEvent(s, ej, 0));
    }
    if (getenv("MRRR_DEBUG_TASKS")) {
      std::vector<double> hl(ntask);
      d2h(hl.data(), lam, ntask, s);
      std::vector<Node> hnodes(nnodes);
      d2h(hnodes.data(), dnodes, nnodes, s);
      for (int t = 0; t < ntask; ++t) {
        const Node &N = hnodes[tasks[t].node];
        fprintf(stderr, "task %d slot %d node %d col %ld lam %.17g tau %.17g + %.3g sigma %.17g depth %d\n", t,
                tasks[t].slot, tasks[t].node, (long)tasks[t].col, hl[t], N.tau_hi, N.tau_lo, N.sigma, N.depth);
      }
    }
    k_output<<<(ntask + 255) / 256, 256, 0, s>>>(dt, ntask, dnodes, lam, 1.0 / scale, w_loc);
    CK(cudaGetLastError());
    g_stats.kernel_launches++;
  }
  });
  finish_w();
  d2h(h_ctr, ctr, 48, s);
  for (int k = 0; k < 16; ++k) g_rqc_hist[k] = (int64_t)h_ctr[32 + k];
  if (tr.on)
    fprintf(stderr, "[mrrr] probes %llu; nudged vector factorizations %llu (why %llu); slowest vector warp: "
            "cycles full %llu rqc %llu solve %llu, max factorizations per warp %llu\n",
            h_ctr[16], h_ctr[10], h_ctr[11], h_ctr[12], h_ctr[13], h_ctr[14], h_ctr[15]);
  if (tr.on)
    fprintf(stderr, "[mrrr] child step max cycles: candidates %llu, probe bwd %llu, probe fwd %llu; "
            "twist+scan %llu; growth %llu\n", h_ctr[18], h_ctr[19], h_ctr[20], h_ctr[21], h_ctr[22]);
  tr.mark("vectors");
  g_stats.ms_vectors = tv.stop();
  g_stats.root_sweeps += h_ctr[0];
  g_stats.safe_resweeps = h_ctr[1];
  g_stats.refine_sweeps = h_ctr[2];
  g_stats.rqc_iters = h_ctr[8];
  g_stats.rqc_fallbacks = h_ctr[9];
  g_stats.vec_nudges = h_ctr[10];
  g_stats.ms_total = tall.stop();
  g_stats.ms_k_root_bisect = kt_root.ms();
  {
    double ms = 0;
    for (auto &e : vec_ev) {
      float v = 0;
      cudaEventSynchronize(e.second);
      cudaEventElapsedTime(&v, e.first, e.second);
      ms += v;
    }
    g_stats.ms_k_vectors = ms;
  }
  if (timeline) {
    cudaStreamSynchronize(s);
    for (size_t i = 0; i < tline.size(); ++i) {
      float v = 0;
      cudaEventElapsedTime(&v, tall.a, tline[i].second);
      fprintf(stderr, "[mrrr timeline] %8.3f ms  tree  %s  (host enqueued it at %.3f ms)\n", v,
              tline[i].first.c_str(), tline_host[i]);
    }
    for (size_t i = 0; i < vec_ev.size(); ++i) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, tall.a, vec_ev[i].first);
      cudaEventElapsedTime(&b, tall.a, vec_ev[i].second);
      fprintf(stderr, "[mrrr timeline] %8.3f ms  piece %zu (level %d) ends %8.3f ms (%.3f ms)\n", a, i,
              vec_ev_level[i], b, b - a);
    }
  }
  g_stats.ms_k_final_refine = kt_fin.ms();
  // bytes this call used: the call arena, the largest level arena, the
  // cluster-step scratch it asked for (the chunks held may be larger: they
  // grow geometrically and are kept for the next call)
  g_stats.workspace_bytes = (int64_t)device_ws(g_ws_call).used + (int64_t)device_ws(g_ws_level).used_peak +
                            (int64_t)cs_scratch_used;
  return 0;
}

int validate(int64_t n, const double *d, const double *e, int range, double vl, double vu,
             int64_t il, int64_t iu, const int64_t *m, const double *w, const double *Z,
             int64_t ldz) {
  if (n < 1) return -1;
  if (!d) return -2;
  if (n > 1 && !e) return -3;
  if (range < 0 || range > 2) return -4;
  if (range == MRRR_RANGE_VALUE) {
    if (!std::isfinite(vl)) return -5;
    if (!std::isfinite(vu) || !(vl < vu)) return -6;
  }
  if (range == MRRR_RANGE_INDEX) {
    if (il < 1 || il > n) return -7;
    if (iu < il || iu > n) return -8;
  }
  if (!m) return -9;
  if (!w) return -10;
  if (Z && ldz < n) return -12;
  if (n > (int64_t)1 << 30) return -1;
  return 0;
}

}  // namespace

extern "C" {

void mrrr_default_opts(mrrr_opts_t *o) {
  o->tol_relgap = 1e-3;
  o->rtol_class = std::ldexp(1.0, -20);
  o->max_depth = 128;
  o->perturb_root = 1;
  o->seed = 0x1205210700000000ULL;
  o->multisection = 4;
  o->grid_factor = 4;
  o->rtol_vec = 0.0;
  o->rqc_max = 10;
  o->shift_strategy = 1;  // DESIGN.md reading 30: interior shift first for clusters of >= 2000 members
  o->scratch_gb = 16.0;
}

// mrrr_negcount: the bisection kernels' Sturm count (projective sweep with
// the qd safe fallback, common.cuh) of a caller-given representation, one
// thread per shift -- the same per-row operations as k_grid / k_refine_warp.
__global__ void k_diag_interleave(const double *D, const double *LLD, int nb, double2 *DL) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) DL[i] = make_double2(D[i], i < nb - 1 ? LLD[i] : 0.0);
}
// The refinement kernels' twisted count (k_refine_warp<M, true>, reading 32)
// on one thread: stationary steps over rows 0 .. r-1, progressive steps over
// rows nb-2 .. r with (D, LLD) swapped, rescales after every 8th step of each
// part, a final rescale, and gamma_r's sign -- the same operations in the
// same order as the warp kernel's lanes, so the same count.
__device__ unsigned negcount_twisted_global(const double2 *__restrict__ DL, int nb, double mu) {
  const int Lf = ((nb - 1) / 32) * 16, Lb = nb - 1 - Lf;
  Sturm f, b;
  sturm_init(f, mu);
  sturm_init(b, mu);
  b.p = __ldg(&DL[nb - 1]).x - mu;
  bool ok = true;
  for (int i = 0; i < Lf; ++i) {
    const double2 v = __ldg(&DL[i]);
    sturm_step(f, v.x, v.y, mu);
    if ((i & 7) == 7) ok &= sturm_rescale(f);
  }
  for (int q = 0; q < Lb; ++q) {
    const double2 v = __ldg(&DL[nb - 2 - q]);
    sturm_step(b, v.y, v.x, mu);
    if ((q & 7) == 7) ok &= sturm_rescale(b);
  }
  ok &= sturm_rescale(f); ok &= sturm_ok(f);
  ok &= sturm_rescale(b); ok &= sturm_ok(b);
  if (!ok || g_force_safe) return negcount_qd_safe(DL, nb, mu);
  const double X = fma(mu, f.q, f.p);
  const double Ng = fma(X, b.q, b.p * f.q);
  const unsigned ng = (Ng != 0.0) ? (((unsigned)(hi32(Ng) ^ hi32(f.q) ^ hi32(b.q))) >> 31) : 0u;
  return f.c + b.c + ng;
}
__global__ void k_diag_negcount(const double2 *DL, int nb, const double *mu, int64_t k, int mode,
                                int64_t *out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= k) return;
  out[q] = mode == 1   ? (int64_t)negcount_qd_safe(DL, nb, mu[q])
           : mode == 2 ? (int64_t)negcount_twisted_global(DL, nb, mu[q])
                       : (int64_t)negcount_global(DL, nb, mu[q], nullptr);
}

__global__ void k_n1(const double *d, double *w, double *Z) {
  w[0] = d[0];
  if (Z) Z[0] = 1.0;
}

// mrrr_stemr after validation; hZ (pinned host, leading dimension hldz) =
// stream Z's column blocks to the host as they complete (mrrr_stemr_host).
int stemr_device(int64_t n, const double *d, const double *e, int range, double vl, double vu,
                 int64_t il, int64_t iu, int64_t *m, double *w, double *Z, int64_t ldz,
                 void *stream, const mrrr_opts_t *opts, double *hZ, int64_t hldz) {
  Problem P;
  P.n = n; P.d = d; P.e = e; P.range = range; P.vl = vl; P.vu = vu; P.il = il; P.iu = iu;
  P.w = w; P.Z = Z; P.ldz = ldz; P.s = (cudaStream_t)stream;
  P.hZ = (n > 1 && Z) ? hZ : nullptr; P.hldz = hldz;
  if (opts) P.o = *opts; else mrrr_default_opts(&P.o);
  if (P.o.rtol_vec != 0.0) return -14;  // oracle-only experiment (reading 10)
  try {
    if (n == 1) {
      double dv;
      CK(cudaMemcpyAsync(&dv, d, sizeof(double), cudaMemcpyDeviceToHost, P.s));
      CK(cudaStreamSynchronize(P.s));
      if (!std::isfinite(dv)) return -2;
      bool in = range != MRRR_RANGE_VALUE || (dv > vl && dv <= vu);
      *m = in ? 1 : 0;
      if (in) {
        k_n1<<<1, 1, 0, P.s>>>(d, w, Z);
        CK(cudaGetLastError());
      }
      CK(cudaStreamSynchronize(P.s));
      return 0;
    }
    auto t0 = std::chrono::steady_clock::now();
    int rc = solve(P, m);
    CK(cudaStreamSynchronize(P.s));
    if (getenv("MRRR_TRACE"))
      fprintf(stderr, "[mrrr] call total (wall)         %8.3f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    return rc;
  } catch (const MrrrError &er) {
    cudaStreamSynchronize(P.s);
    return er.code;
  } catch (const CudaError &ce) {
    cudaGetLastError();
    return ce.e == cudaErrorMemoryAllocation ? MRRR_ERR_NOMEM : MRRR_ERR_CUDA;
  }
}

int mrrr_stemr(int64_t n, const double *d, const double *e, int range, double vl, double vu,
               int64_t il, int64_t iu, int64_t *m, double *w, double *Z, int64_t ldz,
               void *stream, const mrrr_opts_t *opts) {
  int v = validate(n, d, e, range, vl, vu, il, iu, m, w, Z, ldz);
  if (v) return v;
  return stemr_device(n, d, e, range, vl, vu, il, iu, m, w, Z, ldz, stream, opts, nullptr, 0);
}

int mrrr_stemr_host(int64_t n, const double *d, const double *e, int range, double vl,
                    double vu, int64_t il, int64_t iu, int64_t *m, double *w, double *Z,
                    int64_t ldz, void *stream, const mrrr_opts_t *opts) {
  int v = validate(n, d, e, range, vl, vu, il, iu, m, w, Z, ldz);
  if (v) return v;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t k = range == MRRR_RANGE_INDEX ? iu - il + 1 : n;
  double *dd = nullptr, *de = nullptr, *dw = nullptr, *dZ = nullptr;
  int rc = 0;
  auto fail = [&](cudaError_t e) {
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? MRRR_ERR_NOMEM : MRRR_ERR_CUDA;
  };
  cudaError_t ce = cudaSuccess;
  do {
    cudaMemPool_t pool;
    try { pool = lib_pool(); } catch (const CudaError &er) { ce = er.e; break; }
    if ((ce = cudaMallocFromPoolAsync((void **)&dd, n * sizeof(double), pool, s))) break;
    if ((ce = cudaMallocFromPoolAsync((void **)&de, std::max<int64_t>(n - 1, 1) * sizeof(double), pool, s))) break;
    if ((ce = cudaMallocFromPoolAsync((void **)&dw, k * sizeof(double), pool, s))) break;
    if (Z && (ce = cudaMallocFromPoolAsync((void **)&dZ, (size_t)n * k * sizeof(double), pool, s))) break;
    if ((ce = cudaMemcpyAsync(dd, d, n * sizeof(double), cudaMemcpyHostToDevice, s))) break;
    if (n > 1 && (ce = cudaMemcpyAsync(de, e, (n - 1) * sizeof(double), cudaMemcpyHostToDevice, s)))
      break;
    // a pinned Z receives its column blocks while the solve runs (copy
    // stream); a pageable one after the solve
    bool pinned = false;
    if (Z) {
      cudaPointerAttributes pa{};
      if (cudaPointerGetAttributes(&pa, Z) == cudaSuccess) pinned = pa.type == cudaMemoryTypeHost;
      cudaGetLastError();
    }
    rc = stemr_device(n, dd, de, range, vl, vu, il, iu, m, dw, dZ, n, stream, opts, pinned ? Z : nullptr, ldz);
    if (rc) break;
    if (*m > 0) {
      if ((ce = cudaMemcpyAsync(w, dw, *m * sizeof(double), cudaMemcpyDeviceToHost, s))) break;
      if (Z && (!pinned || n == 1) &&
          (ce = cudaMemcpy2DAsync(Z, ldz * sizeof(double), dZ, n * sizeof(double), n * sizeof(double), *m,
                                  cudaMemcpyDeviceToHost, s)))
        break;
    }
    ce = cudaStreamSynchronize(s);
  } while (0);
  for (double *p : {dd, de, dw, dZ})
    if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  if (ce != cudaSuccess) return fail(ce);
  return rc;
}

int mrrr_stemr_dist(int64_t n, const double *d, const double *e, int range, double vl,
                    double vu, int64_t il, int64_t iu, int rank, int nranks,
                    mrrr_allgather_fn allgather, void *allgather_ctx, int64_t *m,
                    const mrrr_opts_t *opts, int64_t *col_begin, int64_t *m_local,
                    double *w_all, double *Z_local, int64_t ldz, void *stream) {
  int v = validate(n, d, e, range, vl, vu, il, iu, m, w_all, Z_local, ldz);
  if (v) return v == -9 ? -13 : (v == -10 ? -17 : (v == -12 ? -19 : v));
  if (nranks < 1) return -10;
  if (rank < 0 || rank >= nranks) return -9;
  if (nranks > 1 && !allgather) return -11;
  if (!col_begin) return -15;
  if (!m_local) return -16;
  Problem P;
  P.n = n; P.d = d; P.e = e; P.range = range; P.vl = vl; P.vu = vu; P.il = il; P.iu = iu;
  P.w = w_all; P.Z = Z_local; P.ldz = ldz; P.s = (cudaStream_t)stream;
  P.rank = rank; P.nranks = nranks; P.allgather = allgather; P.ag_ctx = allgather_ctx;
  P.w_all = w_all;
  if (opts) P.o = *opts; else mrrr_default_opts(&P.o);
  if (P.o.rtol_vec != 0.0) return -14;  // oracle-only experiment (reading 10)
  try {
    if (n == 1) {
      // one eigenpair: rank 0 owns it; w on every rank
      double dv;
      CK(cudaMemcpyAsync(&dv, d, sizeof(double), cudaMemcpyDeviceToHost, P.s));
      CK(cudaStreamSynchronize(P.s));
      if (!std::isfinite(dv)) return -2;
      bool in = range != MRRR_RANGE_VALUE || (dv > vl && dv <= vu);
      *m = in ? 1 : 0;
      *col_begin = 0;
      *m_local = (in && rank == 0) ? 1 : 0;
      if (in) {
        k_n1<<<1, 1, 0, P.s>>>(d, w_all, rank == 0 ? Z_local : nullptr);
        CK(cudaGetLastError());
      }
      CK(cudaStreamSynchronize(P.s));
      return 0;
    }
    int rc = solve(P, m);
    CK(cudaStreamSynchronize(P.s));
    *col_begin = P.col_begin;
    *m_local = P.m_local;
    return rc;
  } catch (const MrrrError &er) {
    cudaStreamSynchronize(P.s);
    return er.code;
  } catch (const CudaError &ce) {
    cudaGetLastError();
    return ce.e == cudaErrorMemoryAllocation ? MRRR_ERR_NOMEM : MRRR_ERR_CUDA;
  }
}

// mrrr_stemr_nccl: mrrr_stemr_dist on an NCCL communicator (SURVEY §8(b)'s
// signature).  NCCL is resolved at run time -- the copy the process has
// already loaded (torch's), else libnccl.so.2 on the loader path -- so the
// library has no link-time dependency on it and the single-GPU entries work
// without it.
namespace {
struct NcclApi {
  // ncclResult_t f(...): 0 = ncclSuccess; ncclDataType_t ncclInt8 = 0
  int (*all_gather)(const void *, void *, size_t, int, void *, void *) = nullptr;
  int (*comm_count)(void *, int *) = nullptr;
  int (*comm_user_rank)(void *, int *) = nullptr;
  int (*comm_cu_device)(void *, int *) = nullptr;
  bool ok = false;
};
const NcclApi &nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.comm_count = (decltype(a.comm_count))dlsym(h, "ncclCommCount");
    a.comm_user_rank = (decltype(a.comm_user_rank))dlsym(h, "ncclCommUserRank");
    a.comm_cu_device = (decltype(a.comm_cu_device))dlsym(h, "ncclCommCuDevice");
    a.ok = a.all_gather && a.comm_count && a.comm_user_rank && a.comm_cu_device;
    return a;
  }();
  return api;
}
int nccl_allgather_cb(void *ctx, const void *send, void *recv, size_t bytes, void *stream) {
  return nccl_api().all_gather(send, recv, bytes, /*ncclInt8*/ 0, ctx, stream) == 0 ? 0 : 1;
}
}  // namespace

int mrrr_stemr_nccl(int64_t n, const double *d, const double *e, int range, double vl,
                    double vu, int64_t il, int64_t iu, void *nccl_comm, int64_t *m,
                    const mrrr_opts_t *opts, int64_t *col_begin, int64_t *m_local,
                    double *w_all, double *Z_local, int64_t ldz, void *stream) {
  if (!nccl_comm) return -9;
  const NcclApi &A = nccl_api();
  if (!A.ok) return MRRR_ERR_COMM;
  int nranks = 0, rank = -1, cdev = -1, dev = -2;
  if (A.comm_count(nccl_comm, &nranks) != 0 || A.comm_user_rank(nccl_comm, &rank) != 0 ||
      A.comm_cu_device(nccl_comm, &cdev) != 0)
    return MRRR_ERR_COMM;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return MRRR_ERR_CUDA; }
  if (dev != cdev) return -9;  // the communicator belongs to another device than the current one
  int rc = mrrr_stemr_dist(n, d, e, range, vl, vu, il, iu, rank, nranks, nccl_allgather_cb, nccl_comm, m,
                           opts, col_begin, m_local, w_all, Z_local, ldz, stream);
  // argument positions of mrrr_stemr_dist -> this entry's (9 comm; 10.. = dist's 13..)
  if (rc <= -13) rc += 3;
  return rc;
}

int mrrr_negcount(int64_t nb, const double *D, const double *LLD, int64_t k, const double *mu,
                  int64_t *count, int mode, void *stream) {
  if (nb < 1 || nb > (int64_t)1 << 30) return -1;
  if (!D) return -2;
  if (nb > 1 && !LLD) return -3;
  if (k < 0) return -4;
  if (k > 0 && !mu) return -5;
  if (k > 0 && !count) return -6;
  if (mode < 0 || mode > 2) return -7;
  if (k == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  double2 *DL = nullptr;
  try {
    set_diag_flags(s);
    cudaError_t e = cudaMallocAsync((void **)&DL, (size_t)nb * sizeof(double2), s);
    if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); return MRRR_ERR_NOMEM; }
    CK(e);
    k_diag_interleave<<<(int)((nb + 255) / 256), 256, 0, s>>>(D, LLD, (int)nb, DL);
    CK(cudaGetLastError());
    k_diag_negcount<<<(int)((k + 127) / 128), 128, 0, s>>>(DL, (int)nb, mu, k, mode, count);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(DL, s));
    CK(cudaStreamSynchronize(s));
    return 0;
  } catch (const CudaError &ce) {
    cudaGetLastError();
    return ce.e == cudaErrorMemoryAllocation ? MRRR_ERR_NOMEM : MRRR_ERR_CUDA;
  }
}

int mrrr_plan_columns(int64_t m, int nranks, const unsigned char *free_cut, int64_t *cuts) {
  if (m < 0) return -1;
  if (nranks < 1) return -2;
  if (m > 0 && !free_cut) return -3;
  if (!cuts) return -4;
  plan_columns(m, nranks, free_cut, cuts);
  return 0;
}

int mrrr_trim_workspace(void) {
  for (auto &w : g_ws_call) w.release();
  for (auto &w : g_ws_level) w.release();
  for (auto &b : g_child_scratch_arr) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr; b.cap = 0;
  }
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto &p : g_pools)
    if (p && cudaMemPoolTrimTo(p, 0) != cudaSuccess) return MRRR_ERR_CUDA;
  return 0;
}

size_t mrrr_workspace_bytes(int64_t n, int64_t k) {
  const double nn = (double)n, kk = (double)std::min(k + 2, n), cap = 16e9;
  const double seg = std::ceil(nn / MRRR_SEG);
  // O(n): scaled d, e, e^2, split flags, root (D, LLD), (LD, LD^2), chain buffers, row->block
  const double fixed = nn * (3 * 8 + 4 + 2 * 16 + 8 + 4 + 4);
  // per slot: j, node, out, active, run end, lo/hi (+ exchange), wl/wu, lambda, fail list,
  // task (24 B), share of a warp item, split-phase state (RqcState + sort keys)
  const double slots = kk * (5 * 4 + 4 * 8 + 8 + 4 + 24 + 1 + 88 + 5 * 4);
  // vector checkpoints: 4 side streams x (piece + 32) columns x 64 B per 16-row segment
  const double ck = std::min(cap, 4.0 * (std::ceil(kk / 4) + 32) * seg * 64.0) + 4.0 * 32 * seg * 64.0;
  // cluster-step scratch: kCSRows rows of n doubles per cluster of a level (<= k / 2 clusters)
  const double cs = std::min(cap, std::floor(kk / 2) * kCSRows * 8.0 * (std::ceil(nn / 8) * 8)) +
                    kCSRows * 8.0 * (std::ceil(nn / 8) * 8);
  return (size_t)(fixed + slots + ck + cs) + ((size_t)64 << 20);  // + per-level lists, headroom
}

const char *mrrr_strerror(int code) {
  switch (code) {
    case 0: return "success";
    case 1: return "root representation not found (definite shift failed after retries)";
    case 2: return "child representation not acceptable (element growth too large)";
    case 3: return "representation tree depth cap exceeded";
    case 4: return "bisection or Rayleigh-quotient iteration did not converge";
    case 5: return "CUDA error";
    case 6: return "out of device memory";
    case 7: return "collective (multi-GPU) error";
    default:
      if (code < 0) return "invalid argument";
      return "unknown error";
  }
}

int mrrr_get_stats(mrrr_stats_t *out) {
  if (!out) return -1;
  *out = g_stats;
  return 0;
}

int mrrr_get_rqc_histogram(int64_t *hist16) {
  if (!hist16) return -1;
  memcpy(hist16, g_rqc_hist, sizeof(g_rqc_hist));
  return 0;
}

const char *mrrr_version(void) { return "mrrr-b200 0.1 (sm_100a)"; }

}  // extern "C"
