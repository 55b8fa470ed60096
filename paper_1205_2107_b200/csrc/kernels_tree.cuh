// kernels_tree.cuh -- prep, split, root representation, root grid, adaptive
// multisection, classification (SURVEY §8(a) rows
// a1-a5; the child representations are in kernels_child.cuh).  Included by
// mrrr.cu (single translation unit).
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

// Warp version of pass 1 (one warp per block): rows of d and e^2 come
// through a cp.async ring of 16-row tiles (lanes 0-15: d_i, 16-31:
// e_{i-1}^2), every lane runs the same chain, lane k keeps row k's t_i and
// rescale, and each tile's values are stored with coalesced writes.  The
// arithmetic is that of k_root_chain (same operations, same order).
constexpr int kRCT = 32, kRCRing = 6;  // 32-row tiles: one definiteness check per 32 rows
__global__ void __launch_bounds__(32) k_root_chain_warp(const double *__restrict__ ds,
                                                        const double *__restrict__ es2, Block *blocks,
                                                        int nblocks, double tnrm_scaled, double *tbuf,
                                                        int *sbuf, double *sigma_out, int *fail) {
  __shared__ double rD[kRCRing][kRCT], rE[kRCRing][kRCT];
  const int b = blockIdx.x, lane = threadIdx.x;
  if (b >= nblocks) return;
  const Block B = blocks[b];
  if (B.nb < 2 || B.slot1 <= B.slot0) { if (lane == 0) sigma_out[b] = 0.0; return; }
  const double *dr = ds + B.row0;
  const double *er = es2 + B.row0;  // er[i-1] = e_{i-1}^2 of the block
  const int nb = B.nb, ntile = (nb + kRCT - 1) / kRCT;
  auto issue = [&](int t) {
    const int slot = t % kRCRing, k = lane, row = t * kRCT + k;
    if (t < ntile && row < nb) {
      __pipeline_memcpy_async(&rD[slot][k], &dr[row], sizeof(double));
      if (row > 0) __pipeline_memcpy_async(&rE[slot][k], &er[row - 1], sizeof(double));
    }
    __pipeline_commit();
  };
  double delta = 4.0 * kEps * tnrm_scaled;
  for (int attempt = 0; attempt <= 6; ++attempt) {
    const double sigma = B.side > 0 ? B.gl - delta : B.gu + delta;
    double tm1 = 1.0, tm2 = 0.0;
    double tlast = 1.0;  // t of the previous tile's last row (t_{-1} = 1)
    bool ok = true;
#pragma unroll
    for (int k = 0; k < kRCRing - 1; ++k) issue(k);
    for (int t = 0; t < ntile; ++t) {
      __pipeline_wait_prior(kRCRing - 2);
      __syncwarp();
      const int slot = t % kRCRing, r0 = t * kRCT, rows = min(kRCT, nb - r0);
      double kt = 0.0;
      int ks = 0;
      // the dependent chain only: t_i = (d_i - sigma) t_{i-1} - e_{i-1}^2 t_{i-2};
      // the definiteness of the tile's rows is checked after it, lane-parallel
      auto row = [&](int k, double di, double b2) {
        const int i = r0 + k;
        const double tt = fma(di - sigma, tm1, -b2 * tm2);
        int sh = 0;
        tm2 = tm1; tm1 = tt;
        if ((i & 7) == 7) {
          const int ee = max_exp(tm1, tm2);
          ok &= ee < 2047 && ee > 0;
          sh = 1023 - min(max(ee, 1), 2045);
          const double f = pow2(sh);
          tm1 *= f; tm2 *= f;
        }
        if (lane == k) { kt = tt; ks = sh; }
      };
      if (rows == kRCT) {
#pragma unroll
        for (int h = 0; h < kRCT; h += 8) {
          double dv[8], bv[8];  // 8 rows in registers before their chain steps
#pragma unroll
          for (int k = 0; k < 8; ++k) { dv[k] = rD[slot][h + k]; bv[k] = (r0 + h + k > 0) ? rE[slot][h + k] : 0.0; }
#pragma unroll
          for (int k = 0; k < 8; ++k) row(h + k, dv[k], bv[k]);
        }
      } else {
        for (int k = 0; k < rows; ++k) row(k, rD[slot][k], (r0 + k > 0) ? rE[slot][k] : 0.0);
      }
      // row r0 + lane: D_i = t_i / t_{i-1} must be finite, non-zero and of the
      // side's sign (the rescale factors are positive: signs are unchanged)
      const double tp = __shfl_up_sync(0xffffffffu, kt, 1);
      const double tprev = lane == 0 ? tlast : tp;
      const bool good = lane >= rows || (kt != 0.0 && isfinite(kt) &&
                                         ((B.side > 0) ? (negbit(kt, tprev) == 0) : (negbit(kt, tprev) == 1)));
      ok &= __all_sync(0xffffffffu, good);
      tlast = __shfl_sync(0xffffffffu, kt, rows - 1);
      if (lane < rows) { tbuf[B.row0 + r0 + lane] = kt; sbuf[B.row0 + r0 + lane] = ks; }
      __syncwarp();
      issue(t + kRCRing - 1);
    }
    __pipeline_wait_prior(0);
    __syncwarp();
    if (ok) { if (lane == 0) sigma_out[b] = sigma; return; }
    delta *= 2.0;
  }
  if (lane == 0) { fail[0] = 1; sigma_out[b] = 0.0; }
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

// ===========================================================================
// Work item of the bisection kernels: a chunk of slots of one node.
struct Work {
  int32_t node;
  int32_t s0, s1;  // slot range
  int32_t pad;
};

// a3 -- root grid: counts of the root representation at G uniformly spaced
// points x_g = lo0 + (hi0 - lo0) g / G, g = g_begin .. g_end-1 within
// [1, G-1] (one CTA handles blockDim.x * M consecutive points; a multi-GPU
// rank evaluates its share of the points).  cnt[g].
template <int M>
__global__ void __launch_bounds__(128) k_grid(const Node *nodes, int node, double lo0, double hi0,
                                              int G, int g_begin, int g_end, int *cnt,
                                              unsigned long long *safe_ctr) {
  __shared__ double2 sm[2 * kTile];
  const Node N = nodes[node];
  double mu[M];
  int g0 = (blockIdx.x * blockDim.x + threadIdx.x) * M + g_begin;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    int g = min(g0 + c, g_end - 1);
    mu[c] = lo0 + (hi0 - lo0) * ((double)g / (double)G);
  }
  unsigned k[M];
  bool ok;
  cta_sweep<M>(N.DL, N.nb, sm, mu, k, ok);
#pragma unroll
  for (int c = 0; c < M; ++c) {
    int g = g0 + c;
    if (g < g_end) {
      unsigned v = k[c];
      if (!ok || g_force_safe) { atomicAdd(safe_ctr, 1ull); v = negcount_qd_safe(N.DL, N.nb, mu[c]); }
      cnt[g] = (int)v;
    }
  }
}

// a3/a5 -- the adaptive multisection per WARP (k_refine_warp): one warp owns up
// to kRWMembers member slots of one node and sweeps the node once per round
// with 32 * M shifts spread over its unconverged members (P = min(32 M / a,
// 64) each: a lone member gains 6 bits per sweep).  Rows come through a
// warp-private shared-memory ring of 16-row tiles filled by cp.async ahead of
// the chains, so warps of different clusters never wait on each other (the
// CTA-wide version spent most of its time in barrier stalls: ncu 9.3 barrier
// stalls per issue).  Invariant N(lo) < j <= N(hi); a member stops when
// hi - lo <= rtol max(|lo|, |hi|) or no double lies strictly inside.  With
// `verify` set (child coordinates, O9.4) a member's first grid includes both
// ends; an end that does not bracket index j is widened by doubling its
// offset from the translated parent interval (plo - wl, phi + wu), and the
// member is narrowed only once both ends bracket j.
constexpr int kRWMembers = 32;  // capacity; a work item holds <= kRWMembers slots
constexpr int kRWT = 16, kRWRing = 6, kRWWarps = 4;

struct RefWarpSmem {
  double2 ring[kRWRing][2 * kRWT];  // SPLIT: [0, 16) the top part's tile, [16, 32) the bottom's
  double lo[kRWMembers], hi[kRWMembers], wl[kRWMembers], wu[kRWMembers];
  double plo[kRWMembers], phi[kRWMembers];
  int j[kRWMembers], state[kRWMembers], act[kRWMembers];
  int cnt[32 * 4];
};

template <int M, bool SPLIT>
__global__ void __launch_bounds__(32 * kRWWarps) k_refine_warp(const Node *nodes, const Work *work, int nwork,
                                                               const int *__restrict__ slot_list,
                                                               const int *__restrict__ slot_j, double *lo_arr,
                                                               double *hi_arr, const double *wlo_arr,
                                                               const double *whi_arr, int verify, double rtol,
                                                               int max_rounds, int *fail,
                                                               unsigned long long *sweeps,
                                                               unsigned long long *safe_ctr,
                                                               double class_tol = 0.0, double early_w = 0.0) {
  static_assert(M >= 1 && M <= 4, "cnt[] is sized for at most 4 shifts per lane");
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
    // shifts: lane l runs C = M (whole sweep) or 2M (SPLIT: lanes l and l^16
    // share the same 2M shifts, l < 16 the top part, l >= 16 the bottom part)
    constexpr int C = SPLIT ? 2 * M : M;
    const int hl = SPLIT ? (lane & 15) : lane;
    double mu[C];
    bool any = false;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int f = hl * C + c;
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
    Sturm st[C];
    bool ok = true;
    if (!SPLIT) {
      // ---- one sweep of the node for the lane's M shifts
#pragma unroll
      for (int c = 0; c < C; ++c) sturm_init(st[c], mu[c]);
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
            double2 v[kRWT];  // the tile's rows in registers before the dependent steps
#pragma unroll
            for (int k = 0; k < kRWT; ++k) v[k] = T[k];
#pragma unroll
            for (int k = 0; k < kRWT; ++k) {
#pragma unroll
              for (int c = 0; c < C; ++c) sturm_step(st[c], v[k].x, v[k].y, mu[c]);
              if ((k & 7) == 7) {
#pragma unroll
                for (int c = 0; c < C; ++c) ok &= sturm_rescale(st[c]);
              }
            }
          } else {
            for (int k = 0; k < rows; ++k) {
              const double2 v = T[k];
#pragma unroll
              for (int c = 0; c < C; ++c) sturm_step(st[c], v.x, v.y, mu[c]);
              if ((k & 7) == 7) {
#pragma unroll
                for (int c = 0; c < C; ++c) ok &= sturm_rescale(st[c]);
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
      for (int c = 0; c < C; ++c) { sturm_last(st[c], Dl); ok &= sturm_ok(st[c]); }
    } else {
      // ---- the count as a twisted factorization at row r (LAPACK dlaneg's
      // form, reading 32): the stationary transform over rows
      // 0 .. r-1 (lanes < 16) and the progressive one over rows nb-2 .. r
      // (lanes >= 16) run at the same time, then
      //   N(mu) = #{D+_i < 0, i < r} + #{D-_i < 0, i > r} + [gamma_r < 0],
      //   gamma_r = s_r + mu + p_r.
      // The progressive step in projective form, p = a/b: u = LLD_i b + a
      // (= D-_i b), a' = D_i a - mu u, b' = u -- the stationary step with
      // (D, LLD) swapped, so both halves run the same instructions.
      const bool fwd = lane < 16;
      const int Lf = ((nb - 1) / (2 * kRWT)) * kRWT;  // r: whole tiles on top
      const int Lb = nb - 1 - Lf;                     // >= Lf rows below
      const int ntf = Lf / kRWT, ntb = (Lb + kRWT - 1) / kRWT;
      const double Dl = __ldg(&N.DL[nb - 1]).x;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        sturm_init(st[c], mu[c]);
        if (!fwd) st[c].p = Dl - mu[c];
      }
      auto issue = [&](int t) {
        if (fwd) {
          if (t < ntf) __pipeline_memcpy_async(&S.ring[t % kRWRing][hl], &N.DL[t * kRWT + hl], sizeof(double2));
        } else {
          const int row = nb - 2 - (t * kRWT + hl);
          if (t < ntb && row >= Lf) {  // stored swapped: (LLD, D)
            double2 *dst = &S.ring[t % kRWRing][kRWT + hl];
            __pipeline_memcpy_async(&dst->x, &N.DL[row].y, sizeof(double));
            __pipeline_memcpy_async(&dst->y, &N.DL[row].x, sizeof(double));
          }
        }
        __pipeline_commit();
      };
      // the sign of each pivot t (= D+ q) goes into a bit mask (one funnel
      // shift per step); a tile's negative pivots are the sign CHANGES of
      // consecutive t (q_i = t_{i-1} up to a positive power of two, q_0 > 0),
      // popc(m ^ (m >> 1)) over its rows -- negbit's count, bit for bit
      unsigned sg[C];
#pragma unroll
      for (int c = 0; c < C; ++c) sg[c] = 0u;
      auto step = [&](int c, double x, double y) {
        const double tt = fma(x, st[c].q, st[c].p);
        sg[c] = __funnelshift_l((unsigned)hi32(tt), sg[c], 1);
        st[c].p = fma(-mu[c], tt, y * st[c].p);
        st[c].q = tt;
      };
#pragma unroll
      for (int k = 0; k < kRWRing - 1; ++k) issue(k);
      for (int t = 0; t < ntb; ++t) {
        __pipeline_wait_prior(kRWRing - 2);
        __syncwarp();
        const double2 *T = S.ring[t % kRWRing] + (fwd ? 0 : kRWT);  // (x, y) = (D, LLD) / (LLD, D)
        if (any) {
          if (t < ntf && (t + 1) * kRWT <= Lb) {  // both halves step a whole tile
            double x[kRWT], y[kRWT];
#pragma unroll
            for (int k = 0; k < kRWT; ++k) { const double2 v = T[k]; x[k] = v.x; y[k] = v.y; }
#pragma unroll
            for (int k = 0; k < kRWT; ++k) {
#pragma unroll
              for (int c = 0; c < C; ++c) step(c, x[k], y[k]);
              if ((k & 7) == 7) {
#pragma unroll
                for (int c = 0; c < C; ++c) ok &= sturm_rescale(st[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) st[c].c += __popc((sg[c] ^ (sg[c] >> 1)) & 0xffffu);
          } else {
            const int rows = fwd ? (t < ntf ? kRWT : 0) : min(kRWT, Lb - t * kRWT);
            for (int k = 0; k < rows; ++k) {
              const double x = T[k].x, y = T[k].y;
#pragma unroll
              for (int c = 0; c < C; ++c) step(c, x, y);
              if ((k & 7) == 7) {
#pragma unroll
                for (int c = 0; c < C; ++c) ok &= sturm_rescale(st[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) st[c].c += __popc((sg[c] ^ (sg[c] >> 1)) & ((1u << rows) - 1u));
          }
        }
        __syncwarp();
        issue(t + kRWRing - 1);
      }
      __pipeline_wait_prior(0);
      // normalise both states (max(|p|, |q|) in [1, 2)), then combine at r
#pragma unroll
      for (int c = 0; c < C; ++c) { ok &= sturm_rescale(st[c]); ok &= sturm_ok(st[c]); }
      ok &= __shfl_xor_sync(0xffffffffu, (int)ok, 16) != 0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double a = __shfl_xor_sync(0xffffffffu, st[c].p, 16);
        const double b = __shfl_xor_sync(0xffffffffu, st[c].q, 16);
        const unsigned cb = __shfl_xor_sync(0xffffffffu, st[c].c, 16);
        // gamma_r q b = (s_r + mu) q b + p_r q b, sign against sign(q b)
        const double X = fma(mu[c], st[c].q, st[c].p);
        const double Ng = fma(X, b, a * st[c].q);
        const unsigned ng = (Ng != 0.0) ? (((unsigned)(hi32(Ng) ^ hi32(st[c].q) ^ hi32(b))) >> 31) : 0u;
        st[c].c += cb + ng;
      }
    }
    if (any && (!ok || g_force_safe) && (!SPLIT || lane < 16)) {
      atomicAdd(safe_ctr, 1ull);
#pragma unroll
      for (int c = 0; c < C; ++c) st[c].c = negcount_qd_safe(N.DL, nb, mu[c]);
    }
    if (!SPLIT || lane < 16) {
#pragma unroll
      for (int c = 0; c < C; ++c) S.cnt[hl * C + c] = (int)st[c].c;
    }
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
    // Reading 31 (tree refinement, class_tol > 0): a verified member stops
    // once its bracket is within early_w (relative) and the classification
    // of both its boundaries is decided: lo_{j+1} - hi_j > class_tol * the
    // largest |endpoint| of the two brackets.  Brackets only shrink, so the
    // test then also holds for the final brackets, where k_classify applies
    // it to the midpoints (|mid| <= that bound): the member is a singleton
    // whatever more bits it would get.  Only neighbours in this work item
    // (verified) or the node's ends count -- the decision depends on the
    // item's own data, so every run and every rank takes the same one.
    if (class_tol > 0.0) {
      bool stop = false;
      if (lane < nm && S.state[lane] == 1) {
        const double l = S.lo[lane], h = S.hi[lane];
        const double ml = fmax(fabs(l), fabs(h));
        if (h - l <= early_w * ml) {
          const int sl = Wk.s0 + lane;
          bool left = sl == N.slot0, right = sl + 1 == N.slot1;
          if (!left && lane > 0 && S.state[lane - 1] != 0) {
            const double nl = S.lo[lane - 1], nh = S.hi[lane - 1];
            left = l - nh > class_tol * fmax(ml, fmax(fabs(nl), fabs(nh)));
          }
          if (!right && lane + 1 < nm && S.state[lane + 1] != 0) {
            const double nl = S.lo[lane + 1], nh = S.hi[lane + 1];
            right = nl - h > class_tol * fmax(ml, fmax(fabs(nl), fabs(nh)));
          }
          stop = left && right;
        }
      }
      __syncwarp();
      if (stop) S.state[lane] = 2;
      __syncwarp();
    }
  }
  if (lane == 0) {
    atomicAdd(sweeps, (unsigned long long)rounds * SH);
    atomicAdd(&g_rw_hist[min(rounds, 63)], 1u);
  }
  if (lane < nm) {
    const int sl = slot_list ? slot_list[Wk.s0 + lane] : Wk.s0 + lane;
    lo_arr[sl] = S.lo[lane]; hi_arr[sl] = S.hi[lane];
    if (S.state[lane] != 2) fail[0] = 1;
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

}  // namespace mrrr
