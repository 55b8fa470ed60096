// kernels_tree.cuh -- prep, root representation, bisection/multisection,
// classification, child representations (SURVEY §8(a)
// rows a1-a5).  Included by mrrr.cu (single translation unit).
#pragma once
#include <cuda_pipeline.h>

#include "common.cuh"

namespace mrrr {

// ===========================================================================
// a1 -- norms, Gershgorin bounds, power-of-two scaling, split
// One CTA of 1024 threads.  hdr: [0] tnrm (unscaled), [1] scale (2^k),
// [2] gl (scaled), [3] gu (scaled); split flags written as int per row.
// ===========================================================================
__global__ void k_prep(const double *__restrict__ d, const double *__restrict__ e, int64_t n,
                       double *__restrict__ ds, double *__restrict__ es, double *__restrict__ es2,
                       int *__restrict__ brk, double *__restrict__ hdr) {
  __shared__ double red[3][32];
  double tn = 0, lo = CUDART_INF, hi = -CUDART_INF;
  int badd = 0, bade = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double r = 0;
    if (i > 0) r += fabs(e[i - 1]);
    if (i < n - 1) { r += fabs(e[i]); bade |= !isfinite(e[i]); }
    double di = d[i];
    badd |= !isfinite(di);
    tn = fmax(tn, r + fabs(di));
    lo = fmin(lo, di - r);
    hi = fmax(hi, di + r);
  }
  for (int o = 16; o; o >>= 1) {
    tn = fmax(tn, __shfl_xor_sync(0xffffffff, tn, o));
    lo = fmin(lo, __shfl_xor_sync(0xffffffff, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffff, hi, o));
  }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { red[0][w] = tn; red[1][w] = lo; red[2][w] = hi; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    tn = l < nw ? red[0][l] : 0.0;
    lo = l < nw ? red[1][l] : CUDART_INF;
    hi = l < nw ? red[2][l] : -CUDART_INF;
    for (int o = 16; o; o >>= 1) {
      tn = fmax(tn, __shfl_xor_sync(0xffffffff, tn, o));
      lo = fmin(lo, __shfl_xor_sync(0xffffffff, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffff, hi, o));
    }
    if (l == 0) { red[0][0] = tn; red[1][0] = lo; red[2][0] = hi; }
  }
  badd = __syncthreads_or(badd);
  bade = __syncthreads_or(bade);
  tn = red[0][0];
  // exact power-of-two scale so that ||T||_1 in [1, 2)
  int ex = 0;
  double sc = 1.0;
  if (tn > 0) { frexp(tn, &ex); sc = ldexp(1.0, 1 - ex); }
  double thr = kEps * tn;  // split threshold on the unscaled data (reading 1)
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    ds[i] = d[i] * sc;
    if (i < n - 1) {
      double ei = e[i];
      bool sp = fabs(ei) <= thr;
      double es_i = sp ? 0.0 : ei * sc;
      es[i] = es_i;
      es2[i] = es_i * es_i;
      brk[i] = sp;
    }
  }
  if (threadIdx.x == 0) {
    hdr[0] = tn; hdr[1] = sc; hdr[2] = red[1][0] * sc; hdr[3] = red[2][0] * sc;
    hdr[4] = badd ? 1.0 : (bade ? 2.0 : 0.0);
  }
}

// ===========================================================================
// Sturm count on the (scaled, split) T itself: projective three-term form
// t_i = (d_i - x) t_{i-1} - e_{i-1}^2 t_{i-2}; counts sign changes.  Used for
// VALUE / multi-block INDEX range selection.  One thread per (x, block).
// ===========================================================================
__device__ inline unsigned sturm_T_count(const double *ds, const double *es2, int64_t r0, int nb,
                                         double x) {
  double tm1 = 1.0, tm2 = 0.0;
  unsigned c = 0;
  bool ok = true;
  for (int i = 0; i < nb; ++i) {
    double b2 = i > 0 ? es2[r0 + i - 1] : 0.0;
    double t = fma(ds[r0 + i] - x, tm1, -b2 * tm2);
    c += negbit(t, tm1);
    tm2 = tm1; tm1 = t;
    if ((i & 7) == 7) {
      int ee = max_exp(tm1, tm2);
      double f = pow2_scale(min(ee, 2045));
      ok &= ee < 2047;
      tm1 *= f; tm2 *= f;
    }
  }
  if (!ok || !isfinite(tm1)) {
    // safe classic count with a tiny-pivot substitution
    double q = 1.0;
    c = 0;
    for (int i = 0; i < nb; ++i) {
      double b2 = i > 0 ? es2[r0 + i - 1] : 0.0;
      q = (ds[r0 + i] - x) - (i > 0 ? b2 / q : 0.0);
      if (fabs(q) < kTiny) q = -kTiny;
      c += q < 0;
    }
  }
  return c;
}

__global__ void k_sturm_T(const double *ds, const double *es2, const Block *blocks, int nblocks,
                          const double *xs, int nx, int *out /* [nx][nblocks] */) {
  int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nx * nblocks) return;
  int xi = id / nblocks, b = id % nblocks;
  out[id] = (int)sturm_T_count(ds, es2, blocks[b].row0, blocks[b].nb, xs[xi]);
}

// ===========================================================================
// a2 -- root representation L0 D0 L0^T = T - sigma0 I.
// Pass 1 (one thread per block, sequential): projective leading minors
//   t_i = (d_i - sigma) t_{i-1} - e_{i-1}^2 t_{i-2}
// (fma chain only), definiteness check, retries with doubled offset.
// Stores t_i and the power-of-two rescale applied after row i.
// Pass 2 (parallel over rows): D_i = t_i / t_{i-1}, L_i = e_i / D_i, seeded
// (1 + 4 eps u) perturbation (reading 3), LD_i, LLD_i.
// ===========================================================================
__global__ void k_root_chain(const double *__restrict__ ds, const double *__restrict__ es2,
                             Block *blocks, int nblocks, double tnrm_scaled, double *tbuf,
                             int *sbuf, double *sigma_out, int *fail) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  Block B = blocks[b];
  if (B.nb < 2 || B.slot1 <= B.slot0) { sigma_out[b] = 0.0; return; }
  double delta = 4.0 * kEps * tnrm_scaled;
  for (int attempt = 0; attempt <= 6; ++attempt) {
    double sigma = B.side > 0 ? B.gl - delta : B.gu + delta;
    double tm1 = 1.0, tm2 = 0.0;
    bool ok = true;
    const double *dr = ds + B.row0;
    const double *er = es2 + B.row0;  // er[i-1] = e_{i-1}^2 of the block
    auto row = [&](int i, double di, double b2) {
      const int64_t gi = B.row0 + i;
      double t = fma(di - sigma, tm1, -b2 * tm2);
      // definite: D_i = t_i / t_{i-1} has the sign of the side
      bool good = (t != 0.0) && ((B.side > 0) ? (negbit(t, tm1) == 0) : (negbit(t, tm1) == 1));
      ok &= good && isfinite(t);
      tbuf[gi] = t;
      int sh = 0;
      tm2 = tm1; tm1 = t;
      if ((i & 7) == 7) {
        int ee = max_exp(tm1, tm2);
        ok &= ee < 2047 && ee > 0;
        sh = 1023 - min(max(ee, 1), 2045);
        double f = pow2(sh);
        tm1 *= f; tm2 *= f;
      }
      sbuf[gi] = sh;
    };
    // rows prefetched one group ahead, ping-pong buffers (in-order issue: a
    // load's first use stalls)
    constexpr int G = 8;
    const int ng = B.nb / G;
    double dx[G], dy[G], ex[G], ey[G];
    auto ld = [&](int i, double (&dd)[G], double (&ee)[G]) {
#pragma unroll
      for (int k = 0; k < G; ++k) { dd[k] = __ldg(&dr[i + k]); ee[k] = (i + k > 0) ? __ldg(&er[i + k - 1]) : 0.0; }
    };
    int m = 0;
    if (ng > 0) {
      ld(0, dx, ex);
      for (; m + 1 < ng; m += 2) {
        const int i = G * m;
        if (i + kPfDist < B.nb) { prefetch_l2(&dr[i + kPfDist]); prefetch_l2(&er[i + kPfDist]); }
        ld(i + G, dy, ey);
#pragma unroll
        for (int k = 0; k < G; ++k) row(i + k, dx[k], ex[k]);
        if (m + 2 < ng) ld(i + 2 * G, dx, ex);
#pragma unroll
        for (int k = 0; k < G; ++k) row(i + G + k, dy[k], ey[k]);
      }
      if (m < ng) {
#pragma unroll
        for (int k = 0; k < G; ++k) row(G * m + k, dx[k], ex[k]);
      }
    }
    for (int i = G * ng; i < B.nb; ++i) row(i, __ldg(&dr[i]), i > 0 ? __ldg(&er[i - 1]) : 0.0);
    if (ok) { sigma_out[b] = sigma; return; }
    delta *= 2.0;
  }
  fail[0] = 1;
  sigma_out[b] = 0.0;
}

__global__ void k_root_finish(const double *__restrict__ ds, const double *__restrict__ es,
                              const Block *blocks, const int *__restrict__ row_block, int64_t n,
                              const double *__restrict__ tbuf, const int *__restrict__ sbuf,
                              const double *__restrict__ sigma_b, int perturb, uint64_t seed,
                              double2 *__restrict__ DL, double2 *__restrict__ LDv) {
  int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= n) return;
  int b = row_block[gi];
  Block B = blocks[b];
  if (B.nb < 2 || B.slot1 <= B.slot0) {
    DL[gi] = make_double2(ds[gi], 0.0);
    LDv[gi] = make_double2(0.0, 0.0);
    return;
  }
  int i = (int)(gi - B.row0);
  // D_i = t_i / t_{i-1}, with t_{i-1} brought to t_i's scale
  double ti = tbuf[gi];
  double tp = (i > 0) ? tbuf[gi - 1] * pow2(sbuf[gi - 1]) : 1.0;
  double D = ti / tp;
  double Lc = 0.0;
  if (i < B.nb - 1) {
    // L_i = e_i / D_i needs D_i (this row); computed here for row i
    Lc = es[gi] / D;
  }
  if (perturb) {
    D = __dmul_rn(D, __dadd_rn(1.0, __dmul_rn(4.0 * kEps, perturb_u(seed, gi, 0))));
    if (i < B.nb - 1) Lc = __dmul_rn(Lc, __dadd_rn(1.0, __dmul_rn(4.0 * kEps, perturb_u(seed, gi, 1))));
  }
  double LD = Lc * D, LLD = Lc * LD;
  DL[gi] = make_double2(D, LLD);
  LDv[gi] = make_double2(LD, LD * LD);
}

// ===========================================================================
// Smem-tiled Sturm sweep of one node by a whole CTA.  Every thread evaluates
// M shifts (independent chains, ILP).  Rows of (D, LLD) are staged through a
// double-buffered shared-memory tile with cp.async and read as warp
// broadcasts.  All threads of the CTA must call it.
// ===========================================================================
constexpr int kTile = 256;  // rows per smem tile (4 KB)

template <int M>
__device__ __forceinline__ void tile_steps(const double2 *__restrict__ t, int rows,
                                           const double (&mu)[M], Sturm (&s)[M], bool &ok) {
  int r = 0;
  for (; r + 8 <= rows; r += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double2 v = t[r + k];
#pragma unroll
      for (int c = 0; c < M; ++c) sturm_step(s[c], v.x, v.y, mu[c]);
    }
#pragma unroll
    for (int c = 0; c < M; ++c) ok &= sturm_rescale(s[c]);
  }
  for (; r < rows; ++r) {
    double2 v = t[r];
#pragma unroll
    for (int c = 0; c < M; ++c) sturm_step(s[c], v.x, v.y, mu[c]);
  }
}

template <int M>
__device__ void cta_sweep(const double2 *__restrict__ DL, int nb, double2 *sm, const double (&mu)[M],
                          unsigned (&cnt)[M], bool &ok) {
  Sturm s[M];
#pragma unroll
  for (int c = 0; c < M; ++c) sturm_init(s[c], mu[c]);
  ok = true;
  const int body = nb - 1;  // rows 0..nb-2 carry LLD; row nb-1 is the last pivot
  const int ntiles = (body + kTile - 1) / kTile;
  auto load = [&](int tile, int buf) {
    int base = tile * kTile;
    int rows = min(kTile, body - base);
    for (int r = threadIdx.x; r < rows; r += blockDim.x)
      __pipeline_memcpy_async(&sm[buf * kTile + r], &DL[base + r], sizeof(double2));
    __pipeline_commit();
  };
  if (ntiles > 0) load(0, 0);
  for (int tile = 0; tile < ntiles; ++tile) {
    int buf = tile & 1;
    if (tile + 1 < ntiles) {
      load(tile + 1, buf ^ 1);
      __pipeline_wait_prior(1);
    } else {
      __pipeline_wait_prior(0);
    }
    __syncthreads();
    int rows = min(kTile, body - tile * kTile);
    tile_steps<M>(sm + buf * kTile, rows, mu, s, ok);
    __syncthreads();
  }
  double Dl = __ldg(&DL[nb - 1]).x;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    sturm_last(s[c], Dl);
    ok &= sturm_ok(s[c]);
    cnt[c] = s[c].c;
  }
}

// As cta_sweep, but a warp whose lanes carry no shift (`work` false for the
// whole warp) only helps stage the tiles and skips the arithmetic.
template <int M>
__device__ void cta_sweep_masked(const double2 *__restrict__ DL, int nb, double2 *sm,
                                 const double (&mu)[M], unsigned (&cnt)[M], bool &ok, bool work) {
  Sturm s[M];
#pragma unroll
  for (int c = 0; c < M; ++c) sturm_init(s[c], mu[c]);
  ok = true;
  const int body = nb - 1;
  const int ntiles = (body + kTile - 1) / kTile;
  auto load = [&](int tile, int buf) {
    int base = tile * kTile;
    int rows = min(kTile, body - base);
    for (int r = threadIdx.x; r < rows; r += blockDim.x)
      __pipeline_memcpy_async(&sm[buf * kTile + r], &DL[base + r], sizeof(double2));
    __pipeline_commit();
  };
  if (ntiles > 0) load(0, 0);
  for (int tile = 0; tile < ntiles; ++tile) {
    int buf = tile & 1;
    if (tile + 1 < ntiles) {
      load(tile + 1, buf ^ 1);
      __pipeline_wait_prior(1);
    } else {
      __pipeline_wait_prior(0);
    }
    __syncthreads();
    if (work) tile_steps<M>(sm + buf * kTile, min(kTile, body - tile * kTile), mu, s, ok);
    __syncthreads();
  }
  double Dl = __ldg(&DL[nb - 1]).x;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    sturm_last(s[c], Dl);
    ok &= sturm_ok(s[c]);
    cnt[c] = s[c].c;
  }
}

// ===========================================================================
// Work item of the bisection kernels: a chunk of slots of one node.
struct Work {
  int32_t node;
  int32_t s0, s1;  // slot range
  int32_t pad;
};

// a3 -- root grid: counts of the root representation at G uniformly spaced
// points x_g = lo0 + (hi0 - lo0) g / G, g = 1..G-1 (one CTA handles
// blockDim.x * M consecutive points).  cnt[g] for g in [1, G-1].
template <int M>
__global__ void __launch_bounds__(128) k_grid(const Node *nodes, int node, double lo0, double hi0,
                                              int G, int *cnt, unsigned long long *safe_ctr) {
  __shared__ double2 sm[2 * kTile];
  const Node N = nodes[node];
  double mu[M];
  int g0 = (blockIdx.x * blockDim.x + threadIdx.x) * M + 1;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    int g = min(g0 + c, G - 1);
    mu[c] = lo0 + (hi0 - lo0) * ((double)g / (double)G);
  }
  unsigned k[M];
  bool ok;
  cta_sweep<M>(N.DL, N.nb, sm, mu, k, ok);
#pragma unroll
  for (int c = 0; c < M; ++c) {
    int g = g0 + c;
    if (g < G) {
      unsigned v = k[c];
      if (!ok) { atomicAdd(safe_ctr, 1ull); v = negcount_qd_safe(N.DL, N.nb, mu[c]); }
      cnt[g] = (int)v;
    }
  }
}

// ===========================================================================
// a3/a5 -- multisection refinement of slot intervals in node coordinates
// until hi - lo <= rtol * max(|lo|, |hi|) or lo, hi have no double between
// them (O7).  Invariant N(lo) < j <= N(hi).  Each thread owns one slot and
// evaluates M shifts per round; the CTA sweeps the node once per round.
// ===========================================================================
template <int M>
__global__ void __launch_bounds__(128) k_bisect(const Node *nodes, const Work *work,
                                                const int *__restrict__ slot_j, double *lo_arr,
                                                double *hi_arr, double rtol, int max_rounds,
                                                unsigned long long *sweeps,
                                                unsigned long long *safe_ctr) {
  __shared__ double2 sm[2 * kTile];
  const Work W = work[blockIdx.x];
  const Node N = nodes[W.node];
  int s = W.s0 + threadIdx.x;
  bool mine = s < W.s1;
  double lo = mine ? lo_arr[s] : 0.0, hi = mine ? hi_arr[s] : 1.0;
  int j = mine ? slot_j[s] : 0;  // block-local 1-based eigen index
  auto conv = [&](double a, double b) {
    double m = 0.5 * (a + b);
    return (b - a <= rtol * fmax(fabs(a), fabs(b))) || !(m > a && m < b);
  };
  bool done = !mine || conv(lo, hi);
  int rounds = 0;
  while (__syncthreads_or(!done) && rounds < max_rounds) {
    double mu[M];
#pragma unroll
    for (int c = 0; c < M; ++c) mu[c] = lo + (hi - lo) * ((double)(c + 1) / (double)(M + 1));
    unsigned k[M];
    bool ok;
    cta_sweep<M>(N.DL, N.nb, sm, mu, k, ok);
    if (!done) {
      if (!ok) {
        atomicAdd(safe_ctr, 1ull);
#pragma unroll
        for (int c = 0; c < M; ++c) k[c] = negcount_qd_safe(N.DL, N.nb, mu[c]);
      }
      double nlo = lo, nhi = hi;
#pragma unroll
      for (int c = 0; c < M; ++c)
        if ((int)k[c] < j && mu[c] > nlo) nlo = mu[c];
#pragma unroll
      for (int c = M - 1; c >= 0; --c)
        if ((int)k[c] >= j && mu[c] > nlo && mu[c] < nhi) nhi = mu[c];
      lo = nlo; hi = nhi;
      done = conv(lo, hi);
    }
    ++rounds;
  }
  if (threadIdx.x == 0) atomicAdd(sweeps, (unsigned long long)rounds * M * (W.s1 - W.s0));
  if (mine) { lo_arr[s] = lo; hi_arr[s] = hi; }
}

// a3/a5 -- adaptive multisection (replaces k_bisect + k_verify on the hot
// path).  One CTA owns up to kRefMax member slots of one node.  Each round the
// CTA sweeps the node once with blockDim.x * M shifts, spread evenly over the
// members that have not converged yet: with a active members each gets
// P = floor(blockDim.x * M / a) shifts, i.e. log2(P + 1) bits per round
// (a lone eigenvalue gains 9 bits per sweep instead of 2.3).  Work item
// slots are W.s0 .. W.s1-1, or slot_list[W.s0 .. W.s1-1] when a list is given.  Counts go to
// shared memory; member i's owner thread then narrows [lo, hi] to the
// neighbouring grid points around index j (invariant N(lo) < j <= N(hi)).
// With `verify` set (child coordinates, O9.4) the member's grid first
// includes both ends; an end that does not bracket j is widened by doubling
// its offset from the translated parent interval (plo - wl, phi + wu) and the
// member is narrowed only once both ends bracket j.
// Stop: hi - lo <= rtol * max(|lo|, |hi|) or no double strictly inside.
constexpr int kRefMax = 128;
constexpr int kPmax = 16;

template <int M>
__global__ void __launch_bounds__(128) k_refine(const Node *nodes, const Work *work,
                                                const int *__restrict__ slot_list,
                                                const int *__restrict__ slot_j, double *lo_arr,
                                                double *hi_arr, const double *wlo_arr,
                                                const double *whi_arr, int verify, double rtol,
                                                int max_rounds, int *fail,
                                                unsigned long long *sweeps,
                                                unsigned long long *safe_ctr) {
  __shared__ double2 sm[2 * kTile];
  __shared__ double m_lo[kRefMax], m_hi[kRefMax], m_wl[kRefMax], m_wu[kRefMax];
  __shared__ double m_plo[kRefMax], m_phi[kRefMax];
  __shared__ int m_j[kRefMax], m_state[kRefMax];  // state: 0 unverified, 1 verified, 2 done
  __shared__ int act[kRefMax];                     // active member ids, compacted
  __shared__ int cnt[128 * M];
  __shared__ int s_na;
  const Work W = work[blockIdx.x];
  const Node N = nodes[W.node];
  const int nm = W.s1 - W.s0;
  const int tid = threadIdx.x, T = blockDim.x, S = T * M;
  auto conv = [&](double a, double b) {
    double m = 0.5 * (a + b);
    return (b - a <= rtol * fmax(fabs(a), fabs(b))) || !(m > a && m < b);
  };
  for (int i = tid; i < nm; i += T) {
    const int sl = slot_list ? slot_list[W.s0 + i] : W.s0 + i;
    m_j[i] = slot_j[sl];
    if (verify) {
      m_plo[i] = lo_arr[sl]; m_phi[i] = hi_arr[sl];
      m_wl[i] = wlo_arr[sl]; m_wu[i] = whi_arr[sl];
      m_lo[i] = m_plo[i] - m_wl[i]; m_hi[i] = m_phi[i] + m_wu[i];
      m_state[i] = 0;
    } else {
      m_lo[i] = lo_arr[sl]; m_hi[i] = hi_arr[sl];
      m_state[i] = conv(m_lo[i], m_hi[i]) ? 2 : 1;
    }
  }
  __syncthreads();
  int rounds = 0;
  for (; rounds < max_rounds; ++rounds) {
    // compact the active members (warp 0; nm <= 128)
    if (tid < 32) {
      int base = 0;
      for (int c0 = 0; c0 < nm; c0 += 32) {
        const int i = c0 + tid;
        const bool a = i < nm && m_state[i] != 2;
        const unsigned b = __ballot_sync(0xffffffffu, a);
        if (a) act[base + __popc(b & ((1u << tid) - 1u))] = i;
        base += __popc(b);
      }
      if (tid == 0) s_na = base;
    }
    __syncthreads();
    const int na = s_na;
    if (na == 0) break;
    // shifts per member: all of the CTA's, up to kPmax (log2(P+1) bits per
    // round; beyond 16 shifts the bits per chain fall below 1/4)
    const int P = min(S / na, kPmax);  // >= M
    double mu[M];
    bool any = false;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const int f = tid * M + c;
      const int ai = f / P, sub = f - ai * P;
      mu[c] = 0.0;
      if (ai < na) {
        const int i = act[ai];
        const double lo = m_lo[i], hi = m_hi[i];
        // unverified: P points over [lo, hi] inclusive; verified: interior
        mu[c] = (m_state[i] == 0) ? lo + (hi - lo) * ((double)sub / (double)(P - 1))
                                  : lo + (hi - lo) * ((double)(sub + 1) / (double)(P + 1));
        if (m_state[i] == 0 && sub == P - 1) mu[c] = hi;
        any = true;
      }
    }
    unsigned k[M];
    bool ok;
    cta_sweep_masked<M>(N.DL, N.nb, sm, mu, k, ok, __any_sync(0xffffffffu, any));
    if (!ok && any) {
      atomicAdd(safe_ctr, 1ull);
#pragma unroll
      for (int c = 0; c < M; ++c) k[c] = negcount_qd_safe(N.DL, N.nb, mu[c]);
    }
#pragma unroll
    for (int c = 0; c < M; ++c) cnt[tid * M + c] = (int)k[c];
    __syncthreads();
    // owners update their member
    for (int ai = tid; ai < na; ai += T) {
      const int i = act[ai];
      const int j = m_j[i];
      const int *cc = cnt + ai * P;
      double lo = m_lo[i], hi = m_hi[i];
      int st = m_state[i];
      if (st == 0) {
        const bool okl = cc[0] <= j - 1, oku = cc[P - 1] >= j;
        if (!okl) { m_wl[i] *= 2.0; lo = m_plo[i] - m_wl[i]; }
        if (!oku) { m_wu[i] *= 2.0; hi = m_phi[i] + m_wu[i]; }
        if (okl && oku) {
          st = 1;
          double nlo = lo, nhi = hi;
          for (int q = 1; q < P - 1; ++q) {
            const double x = lo + (hi - lo) * ((double)q / (double)(P - 1));
            if (cc[q] < j) nlo = fmax(nlo, x);
          }
          for (int q = P - 2; q >= 1; --q) {
            const double x = lo + (hi - lo) * ((double)q / (double)(P - 1));
            if (cc[q] >= j && x > nlo) nhi = fmin(nhi, x);
          }
          lo = nlo; hi = nhi;
        }
      } else {
        double nlo = lo, nhi = hi;
        for (int q = 0; q < P; ++q) {
          const double x = lo + (hi - lo) * ((double)(q + 1) / (double)(P + 1));
          if (cc[q] < j) nlo = fmax(nlo, x);
        }
        for (int q = P - 1; q >= 0; --q) {
          const double x = lo + (hi - lo) * ((double)(q + 1) / (double)(P + 1));
          if (cc[q] >= j && x > nlo) nhi = fmin(nhi, x);
        }
        lo = nlo; hi = nhi;
      }
      if (st == 1 && conv(lo, hi)) st = 2;
      m_lo[i] = lo; m_hi[i] = hi; m_state[i] = st;
    }
    __syncthreads();
  }
  if (tid == 0) atomicAdd(sweeps, (unsigned long long)rounds * S);
  for (int i = tid; i < nm; i += T) {
    const int sl = slot_list ? slot_list[W.s0 + i] : W.s0 + i;
    lo_arr[sl] = m_lo[i]; hi_arr[sl] = m_hi[i];
    if (m_state[i] != 2) fail[0] = 1;
  }
}

// a3/a5 -- the adaptive multisection per WARP (k_refine_warp): one warp owns up
// to kRWMembers member slots of one node and sweeps the node once per round
// with 32 * M shifts spread over its unconverged members (P = min(32 M / a,
// 64) each: a lone member gains 6 bits per sweep).  Rows come through a
// warp-private shared-memory ring of 16-row tiles filled by cp.async ahead of
// the chains, so warps of different clusters never wait on each other (the
// CTA-wide version spent most of its time in barrier stalls: ncu 9.3 barrier
// stalls per issue).  Same arithmetic and update rules as k_refine.
constexpr int kRWMembers = 8;
constexpr int kRWT = 16, kRWRing = 6, kRWWarps = 4;

struct RefWarpSmem {
  double2 ring[kRWRing][kRWT];
  double lo[kRWMembers], hi[kRWMembers], wl[kRWMembers], wu[kRWMembers];
  double plo[kRWMembers], phi[kRWMembers];
  int j[kRWMembers], state[kRWMembers], act[kRWMembers];
  int cnt[32 * 4];
};

template <int M>
__global__ void __launch_bounds__(32 * kRWWarps) k_refine_warp(const Node *nodes, const Work *work, int nwork,
                                                               const int *__restrict__ slot_list,
                                                               const int *__restrict__ slot_j, double *lo_arr,
                                                               double *hi_arr, const double *wlo_arr,
                                                               const double *whi_arr, int verify, double rtol,
                                                               int max_rounds, int *fail,
                                                               unsigned long long *sweeps,
                                                               unsigned long long *safe_ctr) {
  static_assert(M == 4, "cnt[] is sized for 4 shifts per lane");
  __shared__ RefWarpSmem smem[kRWWarps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kRWWarps + wid;
  if (item >= nwork) return;
  RefWarpSmem &S = smem[wid];
  const Work Wk = work[item];
  const Node N = nodes[Wk.node];
  const int nm = Wk.s1 - Wk.s0;
  const int nb = N.nb, body = nb - 1, ntile = (body + kRWT - 1) / kRWT;
  constexpr int SH = 32 * M;
  auto conv = [&](double a, double b) {
    const double m = 0.5 * (a + b);
    return (b - a <= rtol * fmax(fabs(a), fabs(b))) || !(m > a && m < b);
  };
  if (lane < nm) {
    const int sl = slot_list ? slot_list[Wk.s0 + lane] : Wk.s0 + lane;
    S.j[lane] = slot_j[sl];
    if (verify) {
      S.plo[lane] = lo_arr[sl]; S.phi[lane] = hi_arr[sl];
      S.wl[lane] = wlo_arr[sl]; S.wu[lane] = whi_arr[sl];
      S.lo[lane] = S.plo[lane] - S.wl[lane]; S.hi[lane] = S.phi[lane] + S.wu[lane];
      S.state[lane] = 0;
    } else {
      S.lo[lane] = lo_arr[sl]; S.hi[lane] = hi_arr[sl];
      S.state[lane] = conv(S.lo[lane], S.hi[lane]) ? 2 : 1;
    }
  }
  __syncwarp();
  int rounds = 0;
  for (; rounds < max_rounds; ++rounds) {
    const bool a = lane < nm && S.state[lane] != 2;
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    const int na = __popc(bal);
    if (na == 0) break;
    if (a) S.act[__popc(bal & ((1u << lane) - 1u))] = lane;
    __syncwarp();
    const int P = min(SH / na, 64);
    double mu[M];
    bool any = false;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const int f = lane * M + c;
      const int ai = f / P, sub = f - ai * P;
      mu[c] = 0.0;
      if (ai < na) {
        const int i = S.act[ai];
        const double l = S.lo[i], h = S.hi[i];
        mu[c] = (S.state[i] == 0) ? l + (h - l) * ((double)sub / (double)(P - 1))
                                  : l + (h - l) * ((double)(sub + 1) / (double)(P + 1));
        if (S.state[i] == 0 && sub == P - 1) mu[c] = h;
        any = true;
      }
    }
    // ---- one sweep of the node for the lane's M shifts
    Sturm st[M];
#pragma unroll
    for (int c = 0; c < M; ++c) sturm_init(st[c], mu[c]);
    bool ok = true;
    auto issue = [&](int t) {
      const int row = t * kRWT + lane;
      if (lane < kRWT && t < ntile && row < body)
        __pipeline_memcpy_async(&S.ring[t % kRWRing][lane], &N.DL[row], sizeof(double2));
      __pipeline_commit();
    };
#pragma unroll
    for (int k = 0; k < kRWRing - 1; ++k) issue(k);
    for (int t = 0; t < ntile; ++t) {
      __pipeline_wait_prior(kRWRing - 2);
      __syncwarp();
      const double2 *T = S.ring[t % kRWRing];
      const int rows = min(kRWT, body - t * kRWT);
      if (any) {
        if (rows == kRWT) {
#pragma unroll
          for (int k = 0; k < kRWT; ++k) {
            const double2 v = T[k];
#pragma unroll
            for (int c = 0; c < M; ++c) sturm_step(st[c], v.x, v.y, mu[c]);
            if ((k & 7) == 7) {
#pragma unroll
              for (int c = 0; c < M; ++c) ok &= sturm_rescale(st[c]);
            }
          }
        } else {
          for (int k = 0; k < rows; ++k) {
            const double2 v = T[k];
#pragma unroll
            for (int c = 0; c < M; ++c) sturm_step(st[c], v.x, v.y, mu[c]);
            if ((k & 7) == 7) {
#pragma unroll
              for (int c = 0; c < M; ++c) ok &= sturm_rescale(st[c]);
            }
          }
        }
      }
      __syncwarp();
      issue(t + kRWRing - 1);
    }
    __pipeline_wait_prior(0);
    const double Dl = __ldg(&N.DL[nb - 1]).x;
#pragma unroll
    for (int c = 0; c < M; ++c) { sturm_last(st[c], Dl); ok &= sturm_ok(st[c]); }
    if (any && !ok) {
      atomicAdd(safe_ctr, 1ull);
#pragma unroll
      for (int c = 0; c < M; ++c) st[c].c = negcount_qd_safe(N.DL, nb, mu[c]);
    }
#pragma unroll
    for (int c = 0; c < M; ++c) S.cnt[lane * M + c] = (int)st[c].c;
    __syncwarp();
    // ---- owners update their member (lane ai < na owns active member act[ai])
    if (lane < na) {
      const int i = S.act[lane];
      const int jj = S.j[i];
      const int *cc = S.cnt + lane * P;
      double l = S.lo[i], h = S.hi[i];
      int stt = S.state[i];
      if (stt == 0) {
        const bool okl = cc[0] <= jj - 1, oku = cc[P - 1] >= jj;
        if (!okl) { S.wl[i] *= 2.0; l = S.plo[i] - S.wl[i]; }
        if (!oku) { S.wu[i] *= 2.0; h = S.phi[i] + S.wu[i]; }
        if (okl && oku) {
          stt = 1;
          double nl = l, nh = h;
          for (int q = 1; q < P - 1; ++q) {
            const double x = l + (h - l) * ((double)q / (double)(P - 1));
            if (cc[q] < jj) nl = fmax(nl, x);
          }
          for (int q = P - 2; q >= 1; --q) {
            const double x = l + (h - l) * ((double)q / (double)(P - 1));
            if (cc[q] >= jj && x > nl) nh = fmin(nh, x);
          }
          l = nl; h = nh;
        }
      } else {
        double nl = l, nh = h;
        for (int q = 0; q < P; ++q) {
          const double x = l + (h - l) * ((double)(q + 1) / (double)(P + 1));
          if (cc[q] < jj) nl = fmax(nl, x);
        }
        for (int q = P - 1; q >= 0; --q) {
          const double x = l + (h - l) * ((double)(q + 1) / (double)(P + 1));
          if (cc[q] >= jj && x > nl) nh = fmin(nh, x);
        }
        l = nl; h = nh;
      }
      if (stt == 1 && conv(l, h)) stt = 2;
      S.lo[i] = l; S.hi[i] = h; S.state[i] = stt;
    }
    __syncwarp();
  }
  if (lane == 0) atomicAdd(sweeps, (unsigned long long)rounds * SH);
  if (lane < nm) {
    const int sl = slot_list ? slot_list[Wk.s0 + lane] : Wk.s0 + lane;
    lo_arr[sl] = S.lo[lane]; hi_arr[sl] = S.hi[lane];
    if (S.state[lane] != 2) fail[0] = 1;
  }
}

// a5 -- bracket verification in child coordinates (O9.4): counts at lo and
// hi; an end that does not bracket index j is widened by doubling its offset
// from the parent interval until it does.
__global__ void __launch_bounds__(128) k_verify(const Node *nodes, const Work *work,
                                                const int *__restrict__ slot_j, double *lo_arr,
                                                double *hi_arr, const double *wlo_arr,
                                                const double *whi_arr, int *fail,
                                                unsigned long long *sweeps,
                                                unsigned long long *safe_ctr) {
  __shared__ double2 sm[2 * kTile];
  const Work W = work[blockIdx.x];
  const Node N = nodes[W.node];
  int s = W.s0 + threadIdx.x;
  bool mine = s < W.s1;
  double lo = 0.0, hi = 1.0, wl = 0.0, wu = 0.0, plo = 0.0, phi = 0.0;
  int j = 0;
  if (mine) {
    plo = lo_arr[s]; phi = hi_arr[s];  // parent-coordinate bracket minus sigma, unwidened
    wl = wlo_arr[s]; wu = whi_arr[s];
    lo = plo - wl; hi = phi + wu;
    j = slot_j[s];
  }
  bool done = !mine;
  int rounds = 0;
  while (__syncthreads_or(!done) && rounds < 200) {
    double mu[2] = {lo, hi};
    unsigned k[2];
    bool ok;
    cta_sweep<2>(N.DL, N.nb, sm, mu, k, ok);
    if (!done) {
      if (!ok) {
        atomicAdd(safe_ctr, 1ull);
        k[0] = negcount_qd_safe(N.DL, N.nb, lo);
        k[1] = negcount_qd_safe(N.DL, N.nb, hi);
      }
      bool okl = (int)k[0] <= j - 1, oku = (int)k[1] >= j;
      if (!okl) { wl *= 2.0; lo = plo - wl; }
      if (!oku) { wu *= 2.0; hi = phi + wu; }
      done = okl && oku;
    }
    ++rounds;
  }
  if (threadIdx.x == 0) atomicAdd(sweeps, (unsigned long long)rounds * 2 * (W.s1 - W.s0));
  if (mine) {
    if (!done) fail[0] = 1;
    lo_arr[s] = lo; hi_arr[s] = hi;
  }
}

// ===========================================================================
// a4 -- classification by relative gap (O8).  For consecutive
// slots s, s+1 of the same node: boundary iff
//   lo_{s+1} - hi_s > tol * max(|mid_s|, |mid_{s+1}|);
// the last slot of a node always ends a run.  flag[s] = 1 iff a run ends at s.
// ===========================================================================
__global__ void k_classify(const int *__restrict__ slot_node, const double *__restrict__ lo,
                           const double *__restrict__ hi, const int *__restrict__ active,
                           int nslots, double tol, int *__restrict__ run_end) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  if (!active[s]) { run_end[s] = 1; return; }
  int f = 1;
  if (s + 1 < nslots && active[s + 1] && slot_node[s + 1] == slot_node[s]) {
    double g = lo[s + 1] - hi[s];
    double m0 = 0.5 * (lo[s] + hi[s]), m1 = 0.5 * (lo[s + 1] + hi[s + 1]);
    f = g > tol * fmax(fabs(m0), fabs(m1));
  }
  run_end[s] = f;
}

// ===========================================================================
// a5 -- child representation by the stationary transform
// L+ D+ L+^T = L D L^T - sigma I, projective form:
//   t_i = D_i q + p (= D+_i q), p' = LLD_i p - sigma t, q' = t.
// The child keeps the block's off-diagonals LD_i (= L+_i D+_i exactly in
// exact arithmetic) and stores (D+_i, LLD+_i = LD_i^2 / D+_i).
// k_cand: growth of the six candidate shifts (offsets 1, 2, 4 beyond each
// cluster end, order L1 R1 L2 R2 L4 R4): raw max |D+| and the
// eigenvector-weighted growth max over the parent's two end vectors z_L, z_R
// of sum |D+_i| z_i^2 / ||z||^2 (reading 9, amended).
// ===========================================================================
struct Cand {
  double sigma;
  double raw;  // max |D+_i| (inf if not finite)
  double wgt;  // max_{z in {z_L, z_R}} sum |D+_i| z_i^2 / ||z||^2 (inf if not finite / no z)
  int32_t cluster;
  int32_t which;  // 0..5 = (mult index) * 2 + (0 left, 1 right)
};

__global__ void k_cand(const Node *nodes, const int *cl_parent, const int *cl_s0, const int *cl_s1,
                       const double *__restrict__ lo, const double *__restrict__ hi, int ncl,
                       const double *__restrict__ zbuf, int64_t zstride, double rtol, Cand *cand) {
  int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= ncl * 6) return;
  int c = id / 6, which = id % 6;
  const Node P = nodes[cl_parent[c]];
  int s0 = cl_s0[c], s1 = cl_s1[c] - 1;
  double mult = (double)(1 << (which >> 1));
  double sigma;
  if ((which & 1) == 0) {
    // offset unit (reading 8 amended): >= 2 rtol_c |lambda|, independent of
    // how far below rtol_c the bracket converged
    double dl = fmax(fmax(2.0 * (hi[s0] - lo[s0]), 2.0 * rtol * fabs(lo[s0])), 4.0 * kEps * fabs(lo[s0]));
    sigma = lo[s0] - mult * dl;
  } else {
    double dr = fmax(fmax(2.0 * (hi[s1] - lo[s1]), 2.0 * rtol * fabs(hi[s1])), 4.0 * kEps * fabs(hi[s1]));
    sigma = hi[s1] + mult * dr;
  }
  const double2 *DL = P.DL;
  const double *zl = zbuf ? zbuf + (int64_t)(2 * c) * zstride : nullptr;
  const double *zr = zbuf ? zbuf + (int64_t)(2 * c + 1) * zstride : nullptr;
  double p = -sigma, q = 1.0, g = 0.0, nl = 0.0, dnl = 0.0, nr = 0.0, dnr = 0.0;
  bool fin = true;
  const int nb = P.nb;
  auto row = [&](int i, const double2 &v, double a, double b) {
    double t = fma(v.x, q, p);
    double dp = t / q;  // D+_i (off the recurrence chain)
    fin &= isfinite(dp) && dp != 0.0;
    double adp = fabs(dp);
    g = fmax(g, adp);
    nl = fma(adp, a * a, nl); dnl = fma(a, a, dnl);
    nr = fma(adp, b * b, nr); dnr = fma(b, b, dnr);
    if (i < nb - 1) { p = fma(-sigma, t, v.y * p); q = t; }
    if ((i & 7) == 7) {
      int ee = max_exp(p, q);
      fin &= ee < 2047;
      double f = pow2_scale(min(ee, 2045));
      p *= f; q *= f;
    }
  };
  if (zl) {
    // rows and both probe vectors prefetched one group ahead (ping-pong)
    constexpr int G = 4;
    const int ng = nb / G;
    double2 vx[G], vy[G];
    double ax[G], ay[G], bx[G], by[G];
    auto ld = [&](int i, double2 (&v)[G], double (&a)[G], double (&b)[G]) {
#pragma unroll
      for (int k = 0; k < G; ++k) { v[k] = __ldg(&DL[i + k]); a[k] = __ldg(&zl[i + k]); b[k] = __ldg(&zr[i + k]); }
    };
    int m = 0;
    if (ng > 0) {
      ld(0, vx, ax, bx);
      for (; m + 1 < ng; m += 2) {
        const int i = G * m;
        if (i + kPfDist < nb) {
          prefetch_l2(&DL[i + kPfDist]);
          if ((i & 15) == 0) { prefetch_l2(&zl[i + kPfDist]); prefetch_l2(&zr[i + kPfDist]); }
        }
        ld(i + G, vy, ay, by);
#pragma unroll
        for (int k = 0; k < G; ++k) row(i + k, vx[k], ax[k], bx[k]);
        if (m + 2 < ng) ld(i + 2 * G, vx, ax, bx);
#pragma unroll
        for (int k = 0; k < G; ++k) row(i + G + k, vy[k], ay[k], by[k]);
      }
      if (m < ng) {
#pragma unroll
        for (int k = 0; k < G; ++k) row(G * m + k, vx[k], ax[k], bx[k]);
      }
    }
    for (int i = G * ng; i < nb; ++i) row(i, __ldg(&DL[i]), __ldg(&zl[i]), __ldg(&zr[i]));
  } else {
    stream_rows<8>(DL, 0, nb, [&](int i, const double2 &v) { row(i, v, 0.0, 0.0); });
  }
  Cand C;
  C.sigma = sigma;
  C.raw = fin ? g : CUDART_INF;
  C.wgt = (fin && zl && dnl > 0 && dnr > 0) ? fmax(nl / dnl, nr / dnr) : CUDART_INF;
  C.cluster = c;
  C.which = which;
  cand[id] = C;
}

// Shift choice (O9.3, reading 9 amended): all six candidates;
// (i) some raw growth <= 8 spdiam: the least raw growth among those; (ii) else
// the least raw growth among the candidates with weighted growth <= 64
// spdiam; (iii) else the least raw growth if <= 1e8 spdiam; else error 2.
// Ties: the earlier candidate (order L1 R1 L2 R2 L4 R4).
__global__ void k_pick(const Node *nodes, const int *cl_parent, const Cand *cand, int ncl,
                       double *sigma_out, int *tier_out, int *fail) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  double spd = nodes[cl_parent[c]].spdiam;
  const Cand *C = cand + 6 * c;
  int b1 = -1, b2 = -1, b3 = -1;
  for (int k = 0; k < 6; ++k) {
    double g = C[k].raw;
    if (g <= 8.0 * spd && (b1 < 0 || g < C[b1].raw)) b1 = k;
    if (isfinite(g) && C[k].wgt <= 64.0 * spd && (b2 < 0 || g < C[b2].raw)) b2 = k;
    if (b3 < 0 || g < C[b3].raw) b3 = k;
  }
  int tier = 0, best = b1;
  if (best < 0) { tier = 1; best = b2; }
  if (best < 0) { tier = 3; best = b3; if (!(C[b3].raw <= 1e8 * spd)) best = -1; }
  if (best < 0) {
    sigma_out[c] = 0.0;
    tier_out[c] = 4;
    fail[0] = 1;
    return;
  }
  sigma_out[c] = C[best].sigma;
  tier_out[c] = tier;
}

// Accepted child, pass 1 (one thread per cluster): projective chain, storing
// t_i and the rescale exponent applied after row i (like the root).
__global__ void k_child_chain(const Node *nodes, const int *cl_parent, const double *sigma, int ncl,
                              int64_t stride, double *tbuf, int *sbuf) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  const Node P = nodes[cl_parent[c]];
  double sg = sigma[c];
  double p = -sg, q = 1.0;
  double *tb = tbuf + (int64_t)c * stride;
  int *sb = sbuf + (int64_t)c * stride;
  const int nb = P.nb;
  stream_rows<8>(P.DL, 0, nb, [&](int i, const double2 &v) {
    double t = fma(v.x, q, p);
    tb[i] = t;
    int sh = 0;
    if (i < nb - 1) {
      p = fma(-sg, t, v.y * p);
      q = t;
      if ((i & 7) == 7) {
        int ee = max_exp(p, q);
        sh = 1023 - min(max(ee, 1), 2045);
        double f = pow2(sh);
        p *= f; q *= f;
      }
    }
    sb[i] = sh;
  });
}

// Accepted child, pass 2 (parallel over clusters x rows): D+_i = t_i / t_{i-1}
// (t_{i-1} brought to t_i's scale), LLD+_i = LD_i^2 / D+_i.
__global__ void k_child_finish(const Node *nodes, const int *cl_parent, const int *cl_node, int ncl,
                               int64_t stride, const double *tbuf, const int *sbuf,
                               const double2 *__restrict__ LDv, double2 *out_base, int *fail) {
  int c = blockIdx.y;
  if (c >= ncl) return;
  const Node P = nodes[cl_parent[c]];
  int nb = P.nb;
  const double *tb = tbuf + (int64_t)c * stride;
  const int *sb = sbuf + (int64_t)c * stride;
  double2 *out = out_base + (int64_t)c * stride;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    double tp = (i > 0) ? tb[i - 1] * pow2(sb[i - 1]) : 1.0;
    double Dp = tb[i] / tp;
    double ld2 = (i < nb - 1) ? LDv[P.row0 + i].y : 0.0;
    double lld = (i < nb - 1) ? ld2 / Dp : 0.0;
    if (!isfinite(Dp) || Dp == 0.0 || !isfinite(lld)) fail[0] = 1;
    out[i] = make_double2(Dp, lld);
  }
  (void)cl_node;
}

}  // namespace mrrr
