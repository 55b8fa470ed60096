// kernels_child.cuh -- a5: the cluster step of one tree level (PAPER.md
// L1092-1111), one CTA of five warps per cluster.
//
// Every dependent recurrence the step needs runs AT THE SAME TIME, one per warp:
//   warps 0, 1   the parent's twisted factorization at the cluster's left end
//                eigenvalue (stationary from the top, progressive from the
//                bottom), warps 2, 3 the same at the right end -- the probes
//                whose vectors weight the tier-(ii) growth test (reading 9);
//   warp 4       the six candidate shifts (offsets 1, 2, 4 beyond each end,
//                readings 8 and 9), one per lane, through the projective
//                stationary transform of the parent, storing every D+_i.
// After one chain's latency the rest is parallel over the rows: the twist
// index r = argmin |gamma_i| of each probe, its |z| by log2 scans from r, the
// raw growth max |D+| and the growth weighted by z_L^2 and z_R^2 of every
// candidate (block reductions), the tiered choice, and the chosen child
// (D+_i, LLD+_i = LD_i^2 / D+_i) written with coalesced stores.  (This
// replaces a probe kernel followed by a two-pass child kernel: three chain
// latencies per level instead of one.)
//
// Chain warps: every lane runs the same chain (no divergence) and lane k
// keeps row k's values of a 16-row tile, divides once per tile and stores
// them with one coalesced write; rows come through a per-warp cp.async ring.
// Probe arrays, state before / at row i (kernels_vec.cuh notation):
//   forward   s_i = p_i / q_i,   rho_i = z_i / z_{i+1} = -LD_i q_i / t_i
//   backward  P_i = a_i / b_i,   sig_i = z_{i+1} / z_i = -LD_i b_{i+1} / u_{i+1}
//   gamma_i = s_i + P_i + lambda; z_r = 1; only z_i^2 is used downstream
//   (sum |D+_i| z_i^2 / sum z_i^2), so |z_i| is stored.
#pragma once
#include <cuda_pipeline.h>

#include "common.cuh"

namespace mrrr {

constexpr int kCT = 16;     // rows per tile
#ifndef MRRR_CRING
#define MRRR_CRING 6
#endif
constexpr int kCRing = MRRR_CRING;  // tiles in flight per warp
constexpr int kCSWarps = 5; // 4 probe chains + the candidate warp
constexpr int kNC = 7;      // candidates: 6 at the cluster ends (readings 8, 9) + the interior one (reading 30)
constexpr int kCSRows = kNC + 11; // scratch rows per cluster: t of the candidates, 4 per probe, |z| of 2, q every 8 rows

struct ChainRing {
  double2 rDL[kCRing][kCT];  // (D, LLD)
  double2 rLD[kCRing][kCT];  // (LD, LD^2)
};

constexpr int kCSWarpsAdj = kCSWarps + 4;  // + the probes of the two members next to the interior shift
constexpr int kCSRowsAdj = kCSRows + 10;   // + their 8 probe rows and 2 |z| rows

struct ChildSmem {
  ChainRing ring[kCSWarpsAdj];
  double tq[2][kCT][8];      // candidate tile: t_i, q_i per row and candidate (conflict-free writes)
  double red[kCSWarpsAdj][3 * kNC + 4];  // per-warp partials of the growth reductions
  unsigned okw[kCSWarpsAdj];             // per-warp finiteness masks of the candidates
  double sig[kNC];           // the candidates' shifts
  int has_int;               // the interior candidate exists (reading 30)
  int jint;                  // its gap lies between members jint and jint + 1
  double sig_int;
  double am_v[kCSWarpsAdj];  // per-warp argmin (probes)
  int am_i[kCSWarpsAdj];
  int best, tier, bad;
  double sg;
};

struct ChildArgs {
  const Node *nodes;
  const int *cl_parent, *cl_s0, *cl_s1;
  const double *lo, *hi;       // slot brackets (parent coordinates)
  const double2 *LDv;          // global (LD, LD^2) per row
  int c0, ncl;                 // clusters c0 .. ncl-1 (one CTA each)
  double rtol;
  double *scratch;             // kCSRows * zstride doubles per cluster of the launch
  int64_t zstride;
  double2 *const *pool;        // child c's rows at pool[c] (recycled slots, mrrr.cu)
  double *sigma_out;
  int *tier_out;
  int *fail;
  unsigned long long *ctr;     // [0] probes (twisted factorizations)
  int shift_strategy;          // 1: interior candidate first (reading 30)
  double int_wg;               // the interior candidate's weighted-growth bound (x spdiam)
  const int *cl_list;          // optional: the launch's clusters are cl_list[c0 .. ncl-1]
};

// Issue the rows of tile `tile` into ring slot `slot` (lanes 0-15: (D, LLD),
// lanes 16-31: (LD, LD^2) when needed); always commits a group.
__device__ __forceinline__ void cs_issue(ChainRing &R, const double2 *DL, const double2 *LD, int nb,
                                         int tile, int slot, int lane, bool need_ld) {
  const int k = lane & (kCT - 1);
  if (tile >= 0) {
    const int row = tile * kCT + k;
    if (row < nb) {
      if (lane < kCT) __pipeline_memcpy_async(&R.rDL[slot][k], &DL[row], sizeof(double2));
      else if (need_ld) __pipeline_memcpy_async(&R.rLD[slot][k], &LD[row], sizeof(double2));
    }
  }
  __pipeline_commit();
}

// Stationary chain of a probe: sS[i] = s_i (i < nb), sR[i] = rho_i (i < nb - 1).
__device__ __forceinline__ void cs_probe_fwd(ChainRing &R, const double2 *DL, const double2 *LD, int nb,
                                             double lam, int lane, double *sS, double *sR) {
  const int ntile = (nb + kCT - 1) / kCT;
#pragma unroll
  for (int k = 0; k < kCRing - 1; ++k) cs_issue(R, DL, LD, nb, k < ntile ? k : -1, k, lane, true);
  double p = -lam, q = 1.0;
  for (int c = 0; c < ntile; ++c) {
    __pipeline_wait_prior(kCRing - 2);
    __syncwarp();
    const int slot = c % kCRing, r0 = c * kCT, rows = min(kCT, nb - r0);
    double kp = 0.0, kq = 1.0, kt = 1.0, kld = 0.0;
    auto row = [&](const double2 v, int k, bool last_check) {
      const int i = r0 + k;
      const double tt = fma(v.x, q, p);
      if (lane == k) { kp = p; kq = q; kt = tt; }
      if (!last_check || i < nb - 1) { p = fma(-lam, tt, v.y * p); q = tt; }
      if ((k & 7) == 7) {
        const double f = pow2_scale(min(max(max_exp(p, q), 1), 2045));
        p *= f; q *= f;
      }
    };
    if (lane < kCT) kld = R.rLD[slot][lane].x;
    if (rows == kCT && r0 + kCT < nb) {  // every row of the tile is below nb - 1
#pragma unroll
      for (int h = 0; h < kCT; h += 8) {  // rows in registers, 8 at a time, before the dependent steps
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = R.rDL[slot][h + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) row(v[k], h + k, false);
      }
    } else {
      for (int k = 0; k < rows; ++k) row(R.rDL[slot][k], k, true);
    }
    if (lane < rows) {
      const int i = r0 + lane;
      sS[i] = div_nr(kp, kq);  // probe ratios: weights only
      if (i < nb - 1) sR[i] = -kld * div_nr(kq, kt);
    }
    __syncwarp();
    const int cn = c + kCRing - 1;
    cs_issue(R, DL, LD, nb, cn < ntile ? cn : -1, cn % kCRing, lane, true);
  }
  __pipeline_wait_prior(0);
}

// Progressive chain of a probe: sP[i] = P_i (i < nb), sG[i] = sig_i (i < nb - 1).
__device__ __forceinline__ void cs_probe_bwd(ChainRing &R, const double2 *DL, const double2 *LD, int nb,
                                             double lam, int lane, double *sP, double *sG) {
  const int ntile = (nb + kCT - 1) / kCT;
#pragma unroll
  for (int k = 0; k < kCRing - 1; ++k) cs_issue(R, DL, LD, nb, k < ntile ? ntile - 1 - k : -1, k, lane, true);
  double a = __ldg(&DL[nb - 1]).x - lam, b = 1.0;
  if (lane == 0) sP[nb - 1] = a;
  for (int c = 0; c < ntile; ++c) {
    __pipeline_wait_prior(kCRing - 2);
    __syncwarp();
    const int slot = c % kCRing, r0 = (ntile - 1 - c) * kCT;
    const int top = min(r0 + kCT, nb - 1) - 1;  // rows r0 .. top step (row i from i+1)
    double kb = 1.0, ku = 1.0, ka = 0.0, kld = 0.0;
    auto row = [&](const double2 v, int k) {
      const double u = fma(v.y, b, a);
      const double an = fma(-lam, u, v.x * a);
      if (lane == k) { kb = b; ku = u; ka = an; }
      a = an; b = u;
      if ((k & 7) == 0) {
        const double f = pow2_scale(min(max(max_exp(a, b), 1), 2045));
        a *= f; b *= f;
      }
    };
    if (lane < kCT) kld = R.rLD[slot][lane].x;
    if (top - r0 + 1 == kCT) {
#pragma unroll
      for (int h = kCT - 8; h >= 0; h -= 8) {  // rows in registers, 8 at a time, before the dependent steps
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = R.rDL[slot][h + k];
#pragma unroll
        for (int k = 7; k >= 0; --k) row(v[k], h + k);
      }
    } else {
      for (int k = top - r0; k >= 0; --k) row(R.rDL[slot][k], k);
    }
    if (lane <= top - r0) {
      const int i = r0 + lane;
      sP[i] = div_nr(ka, ku);
      sG[i] = -kld * div_nr(kb, ku);
    }
    __syncwarp();
    const int cn = c + kCRing - 1;
    cs_issue(R, DL, LD, nb, cn < ntile ? ntile - 1 - cn : -1, cn % kCRing, lane, true);
  }
  __pipeline_wait_prior(0);
}

// The candidate chains (lane k < kNC runs shift sig[k]; the other lanes
// repeat lane 0's): TP[k * zstride + i] = t_i (= D+_i q_i) and, every 8 rows,
// QK[k * (zstride / 8) + i / 8] = q_i.  The chain does no division: D+_i =
// t_i / q_i with q_i = t_{i-1} (or QK where the chain rescaled, i % 8 == 0)
// is formed later by all the CTA's threads (cs_dplus) -- the candidate warp
// is the step's critical chain.  Each tile's 16 rows are read into registers
// before the dependent steps.
__device__ __forceinline__ void cs_candidates(ChainRing &R, ChildSmem &S, const double2 *DL, int nb,
                                              double sigma, int lane, double *TP, double *QK, int64_t zstride) {
  const int ntile = (nb + kCT - 1) / kCT;
#pragma unroll
  for (int k = 0; k < kCRing - 1; ++k) cs_issue(R, DL, nullptr, nb, k < ntile ? k : -1, k, lane, false);
  double p = -sigma, q = 1.0;
  const int cand = lane < kNC ? lane : 0;
  double *tp = TP + cand * zstride, *qk = QK + cand * (zstride / 8);
  for (int c = 0; c < ntile; ++c) {
    __pipeline_wait_prior(kCRing - 2);
    __syncwarp();
    const int slot = c % kCRing, r0 = c * kCT, rows = min(kCT, nb - r0);
    auto row = [&](const double2 v, int k, bool last_check) {
      const int i = r0 + k;
      if ((k & 7) == 0 && lane < kNC) qk[i >> 3] = q;
      const double tt = fma(v.x, q, p);
      if (lane < kNC) S.tq[0][k][lane] = tt;
      if (!last_check || i < nb - 1) { p = fma(-sigma, tt, v.y * p); q = tt; }
      if ((k & 7) == 7) {
        const double f = pow2_scale(min(max(max_exp(p, q), 1), 2045));
        p *= f; q *= f;
      }
    };
    if (rows == kCT && r0 + kCT < nb) {  // every row of the tile is below nb - 1
#pragma unroll
      for (int h = 0; h < kCT; h += 8) {  // rows in registers, 8 at a time, before the dependent steps
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = R.rDL[slot][h + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) row(v[k], h + k, false);
      }
    } else {
      for (int k = 0; k < rows; ++k) row(R.rDL[slot][k], k, true);
    }
    __syncwarp();
    // the tile's t values, coalesced: kNC * 16 stores spread over the warp
#pragma unroll
    for (int e = lane; e < kNC * kCT; e += 32) {
      const int cc = e >> 4, k = e & (kCT - 1);
      if (k < rows) TP[cc * zstride + r0 + k] = S.tq[0][k][cc];
    }
    __syncwarp();
    const int cn = c + kCRing - 1;
    cs_issue(R, DL, nullptr, nb, cn < ntile ? cn : -1, cn % kCRing, lane, false);
  }
  __pipeline_wait_prior(0);
}

// D+_i of candidate k from its stored t (cs_candidates): the same quotient
// t_i / q_i the chain's state held, bit for bit.
__device__ __forceinline__ double cs_dplus(const double *TP, const double *QK, int64_t zstride, int k, int i) {
  const double *tp = TP + k * zstride;
  const double q = (i & 7) == 0 ? QK[k * (zstride / 8) + (i >> 3)] : tp[i - 1];
  return div_nr(tp[i], q);
}

// |D+_i| for the growth tests only (reading 9): |t_i| times the hardware
// reciprocal of |q_i| (MUFU.RCP64H, ~2^-22 relative) -- the growth bounds
// (8, 64, 1e8 spdiam) and the least-growth choice do not need the quotient's
// last bits, and the full-precision division per candidate and row was the
// largest cost of the step's reductions.  Non-finite or zero D+ (t or q zero
// or not finite) returns a NaN so that the caller's finiteness test fails.
__device__ __forceinline__ double cs_absdplus_fast(const double *TP, const double *QK, int64_t zstride, int k,
                                                    int i) {
  const double *tp = TP + k * zstride;
  const double q = (i & 7) == 0 ? QK[k * (zstride / 8) + (i >> 3)] : tp[i - 1];
  const double t = tp[i];
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(fabs(q)));
  const bool ok = isfinite(t) && t != 0.0 && isfinite(q) && q != 0.0;
  return ok ? fabs(t) * r : CUDART_NAN;
}

// ADJ = 0: the step of a cluster with the end candidates only (five warps).
// ADJ = 1 (reading 30, clusters of >= 2000 members): also the interior
// candidate, and two more probes (four more warps) at the members next to its
// shift, whose weighted growth the interior child must also pass.
template <int ADJ>
__global__ void __launch_bounds__(32 * (kCSWarps + 4 * ADJ), ADJ ? 1 : 2) k_child_step(ChildArgs A) {
  constexpr int NW = kCSWarps + 4 * ADJ, NP = 2 + 2 * ADJ, ROWS = ADJ ? kCSRowsAdj : kCSRows;
  __shared__ ChildSmem S;
  if (A.c0 + (int)blockIdx.x >= A.ncl) return;
  const int c = A.cl_list ? A.cl_list[A.c0 + blockIdx.x] : A.c0 + (int)blockIdx.x;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const Node P = A.nodes[A.cl_parent[c]];
  const int nb = P.nb;
  const int s0 = A.cl_s0[c], s1 = A.cl_s1[c] - 1;
  const double2 *DL = P.DL, *LD = A.LDv + P.row0;
  const int64_t zs = A.zstride;
  double *base = A.scratch + (int64_t)blockIdx.x * ROWS * zs;
  double *TP = base;                 // the candidates' t
  double *QK = base + (kNC + 10) * zs;  // the candidates' q every 8 rows (zs / 8 each)
  // per probe side: s, P, rho, sig (4 rows) and |z| (1 row); sides 0, 1 the
  // cluster's end members, 2, 3 (ADJ) the members next to the interior shift
  double *pr[4] = {base + kNC * zs, base + (kNC + 4) * zs, base + kCSRows * zs, base + (kCSRows + 4) * zs};
  double *zz[4] = {base + (kNC + 8) * zs, base + (kNC + 9) * zs, base + (kCSRows + 8) * zs, base + (kCSRows + 9) * zs};
  double *zl = zz[0], *zr = zz[1];

  // ---- phase 0 (ADJ): the interior candidate (reading 30) -- the midpoint of
  // the widest conservative gap between consecutive members in the middle
  // half of a cluster of >= 2000 members whose width exceeds 1e-6 spdiam,
  // if that gap exceeds 1e-10 of the members' magnitudes (not a degenerate
  // group); a CTA-wide reduction, ties to the lowest member (the oracle's order)
  if (ADJ) {
    const int mm = s1 - s0 + 1;
    double gb = -CUDART_INF;
    int jbest = -1;
    if (A.shift_strategy == 1 && mm >= 2000 && A.hi[s1] - A.lo[s0] > 1e-6 * P.spdiam) {
      const int ja = s0 + mm / 4, jb = s1 - mm / 4;  // members j in [ja, jb) and j + 1
      for (int j = ja + tid; j < jb; j += 32 * NW) {
        const double gj = A.lo[j + 1] - A.hi[j];
        if (gj > gb) { gb = gj; jbest = j; }
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, gb, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jbest, o);
      if (og > gb || (og == gb && oj >= 0 && (jbest < 0 || oj < jbest))) { gb = og; jbest = oj; }
    }
    if (lane == 0) { S.am_v[wid] = gb; S.am_i[wid] = jbest; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NW; ++w) {
        const double og = S.am_v[w];
        const int oj = S.am_i[w];
        if (og > gb || (og == gb && oj >= 0 && (jbest < 0 || oj < jbest))) { gb = og; jbest = oj; }
      }
      S.has_int = 0; S.jint = s0; S.sig_int = 0.0;
      if (jbest >= 0) {
        const double la = 0.5 * (A.lo[jbest] + A.hi[jbest]), lb = 0.5 * (A.lo[jbest + 1] + A.hi[jbest + 1]);
        if (gb > 1e-10 * fmax(fabs(la), fabs(lb))) {
          S.has_int = 1; S.jint = jbest;
          S.sig_int = 0.5 * (A.hi[jbest] + A.lo[jbest + 1]);
        }
      }
    }
    __syncthreads();
  } else if (tid == 0) {
    S.has_int = 0;
  }
  // probe side of a probe warp (-1: the candidate warp) and its eigenvalue
  const int pside = wid < 4 ? (wid >> 1) : (wid == 4 ? -1 : 2 + ((wid - 5) >> 1));
  const int pw0 = pside < 2 ? 2 * pside : 5 + 2 * (pside - 2);  // first warp of the side
  auto probe_slot = [&](int side) { return side == 0 ? s0 : side == 1 ? s1 : S.jint + (side - 2); };

  // ---- phase 1: the chains (probes: stationary / progressive sweeps; candidates)
  const long long clk_p0 = clock64();
  if (pside >= 0) {
    if (pside < 2 || S.has_int) {
      const int slot = probe_slot(pside);
      const double lam = 0.5 * (A.lo[slot] + A.hi[slot]);
      double *q = pr[pside];
      if (wid == pw0) cs_probe_fwd(S.ring[wid], DL, LD, nb, lam, lane, q, q + 2 * zs);
      else cs_probe_bwd(S.ring[wid], DL, LD, nb, lam, lane, q + zs, q + 3 * zs);
    }
  } else {
    const bool has_int = ADJ && S.has_int;
    const double sig_int = ADJ ? S.sig_int : 0.0;
    const int which = lane < 6 ? lane : 0;
    const double mult = (double)(1 << (which >> 1));
    double sigma;
    if (lane == 6 && has_int) {
      sigma = sig_int;
    } else if ((which & 1) == 0) {
      const double l = A.lo[s0], h = A.hi[s0];
      const double dl = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(l)), 4.0 * kEps * fabs(l));
      sigma = l - mult * dl;
    } else {
      const double l = A.lo[s1], h = A.hi[s1];
      const double dr = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(h)), 4.0 * kEps * fabs(h));
      sigma = h + mult * dr;
    }
    cs_candidates(S.ring[4], S, DL, nb, sigma, lane, TP, QK, zs);
    if (lane < kNC) S.sig[lane] = sigma;
  }
  if (lane == 0) atomicMax(&A.ctr[1 + (wid == 4 ? 1 : (wid & 1) ? 2 : 3)], (unsigned long long)(clock64() - clk_p0));
  __syncthreads();
  const long long clk_p1 = clock64();

  // ---- phase 2: each probe's twist index and |z| (the side's two warps)
  if (pside >= 0 && (pside < 2 || S.has_int)) {
    const int side = pside, gt = tid - 32 * pw0;
    const int pslot = probe_slot(side);
    const double lam = 0.5 * (A.lo[pslot] + A.hi[pslot]);
    const double *sS = pr[side], *sP = pr[side] + zs, *sR = pr[side] + 2 * zs, *sG = pr[side] + 3 * zs;
    double *z = zz[side];
    double bv = CUDART_INF;
    int bi = nb;
#pragma unroll 8
    for (int i = gt; i < nb; i += 64) {
      const double g = fabs(sS[i] + sP[i] + lam);
      if (g < bv) { bv = g; bi = i; }  // ascending i per thread: first minimum kept
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { S.am_v[wid] = bv; S.am_i[wid] = bi; }
    // the two warps of a probe meet here (named barrier per probe)
    asm volatile("bar.sync %0, 64;" ::"r"(1 + side));
    const double v0 = S.am_v[pw0], v1 = S.am_v[pw0 + 1];
    const int i0 = S.am_i[pw0], i1 = S.am_i[pw0 + 1];
    int r = (v1 < v0 || (v1 == v0 && i1 < i0)) ? i1 : i0;
    if (r >= nb) r = nb - 1;  // no finite gamma: any twist (the vector only weights)
    // |z| by a product scan of |ratio| in (mantissa, exponent) form -- m in
    // [1, 2), the exponent a double (exact integers) -- so no product over-
    // or underflows and no transcendental is evaluated.  Blocked warp scan:
    // each step the 32 lanes load 32 consecutive ratios (coalesced, 8 blocks
    // of loads in flight), scan them across the warp and fold in the running
    // carry; one pass writes z.  (Round 1 walked one contiguous run per lane
    // twice: dependent loads, 35 % of the step's samples at level 0.)  A zero
    // or non-finite ratio zeroes the rest of that side (as a log of -inf would).
    const bool up = wid == pw0;         // up: rows r-1 .. 0 from rho; down: rows r+1 .. nb-1 from sig
    const int m = up ? r : nb - 1 - r;  // ratios on this side
    if (up && lane == 0) z[r] = 1.0;
    constexpr double kDead = -1.0e9;    // exponent of a zeroed product
    auto split = [](double x, double &mm, double &ee) {  // |x| = mm 2^ee, mm in [1, 2)
      const long long b = __double_as_longlong(x) & 0x7fffffffffffffffLL;
      const int ex = (int)(b >> 52);
      const bool ok = ex > 0 && ex < 2047;  // normal and finite
      mm = ok ? __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL) : 1.0;
      ee = ok ? (double)(ex - 1023) : kDead;
    };
    auto mul = [](double &mm, double &ee, double m2, double e2) {
      mm *= m2; ee += e2;
      if (mm >= 2.0) { mm *= 0.5; ee += 1.0; }
    };
    auto to_double = [](double mm, double ee) {  // mm 2^ee, 0 below the normal range (weights only)
      if (ee < -1022.0) return 0.0;
      if (ee > 1023.0) return CUDART_INF;
      const int ei = (int)ee;
      return __hiloint2double(__double2hiint(mm) + (ei << 20), __double2loint(mm));
    };
    const double *src = up ? sR + (r - 1) : sG + r;  // x_j = |src[dir * j]|
    const int dir = up ? -1 : 1;
    double *dst = up ? z + (r - 1) : z + (r + 1);
    double cm = 1.0, ce = 0.0;  // carry: product of all earlier blocks
    // each lane multiplies 8 consecutive ratios serially, one warp scan
    // combines the 32 lane products, each lane applies its prefix (5 shuffle
    // steps per 256 rows; the order k_child_step2<0, true> uses too)
    constexpr int kL = 8;
    for (int b0 = 0; b0 < m; b0 += 32 * kL) {
      const int j0 = b0 + lane * kL;
      double xv[kL];
#pragma unroll
      for (int u = 0; u < kL; ++u) xv[u] = j0 + u < m ? src[dir * (j0 + u)] : 1.0;
      double mm[kL], ee[kL];
      double pm = 1.0, pe = 0.0;
#pragma unroll
      for (int u = 0; u < kL; ++u) {
        double im, ie;
        split(xv[u], im, ie);
        if (j0 + u >= m) { im = 1.0; ie = 0.0; }
        mul(pm, pe, im, ie);
        mm[u] = pm; ee[u] = pe;
      }
      double sm = pm, se = pe;
      for (int o = 1; o < 32; o <<= 1) {  // inclusive scan over the 32 lane products
        const double ym = __shfl_up_sync(0xffffffffu, sm, o), ye = __shfl_up_sync(0xffffffffu, se, o);
        if (lane >= o) mul(sm, se, ym, ye);
      }
      double xm = __shfl_up_sync(0xffffffffu, sm, 1), xe = __shfl_up_sync(0xffffffffu, se, 1);
      if (lane == 0) { xm = 1.0; xe = 0.0; }
      mul(xm, xe, cm, ce);
#pragma unroll
      for (int u = 0; u < kL; ++u) {
        double om = mm[u], oe = ee[u];
        mul(om, oe, xm, xe);
        if (j0 + u < m) dst[dir * (j0 + u)] = to_double(om, oe);
      }
      const double tm = __shfl_sync(0xffffffffu, sm, 31), te = __shfl_sync(0xffffffffu, se, 31);
      mul(cm, ce, tm, te);
    }
  }
  __syncthreads();

  __syncthreads();
  if (tid == 0) atomicMax(&A.ctr[5], (unsigned long long)(clock64() - clk_p1));
  const long long clk_p2 = clock64();
  // ---- phase 3: growth of the candidates, raw and weighted (all threads)
  double g[kNC], nl[kNC], nr[kNC], dnl = 0.0, dnr = 0.0;
  double na = 0.0, nbb = 0.0, dna = 0.0, dnb = 0.0;  // ADJ: the interior child against probes 2, 3
  unsigned okm = (1u << kNC) - 1u;
  const bool adj = ADJ && S.has_int;
#pragma unroll
  for (int k = 0; k < kNC; ++k) { g[k] = 0.0; nl[k] = 0.0; nr[k] = 0.0; }
#pragma unroll 2
  for (int i = tid; i < nb; i += 32 * NW) {
    const double a = zl[i], b = zr[i];
    const double a2 = a * a, b2 = b * b;
    dnl += a2; dnr += b2;
#pragma unroll
    for (int k = 0; k < kNC; ++k) {
      const double ad = cs_absdplus_fast(TP, QK, zs, k, i);
      if (!(isfinite(ad) && ad != 0.0)) okm &= ~(1u << k);
      g[k] = fmax(g[k], ad);
      nl[k] = fma(ad, a2, nl[k]);
      nr[k] = fma(ad, b2, nr[k]);
      if (ADJ && k == 6 && adj) {
        const double x = zz[2][i], y = zz[3][i];
        na = fma(ad, x * x, na); nbb = fma(ad, y * y, nbb);
        dna = fma(x, x, dna); dnb = fma(y, y, dnb);
      }
    }
  }
  if (ADJ) {
    for (int o = 16; o; o >>= 1) {
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nbb += __shfl_xor_sync(0xffffffffu, nbb, o);
      dna += __shfl_xor_sync(0xffffffffu, dna, o);
      dnb += __shfl_xor_sync(0xffffffffu, dnb, o);
    }
  }
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int k = 0; k < kNC; ++k) {
      g[k] = fmax(g[k], __shfl_xor_sync(0xffffffffu, g[k], o));
      nl[k] += __shfl_xor_sync(0xffffffffu, nl[k], o);
      nr[k] += __shfl_xor_sync(0xffffffffu, nr[k], o);
    }
    dnl += __shfl_xor_sync(0xffffffffu, dnl, o);
    dnr += __shfl_xor_sync(0xffffffffu, dnr, o);
    okm &= __shfl_xor_sync(0xffffffffu, okm, o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kNC; ++k) {
      S.red[wid][k] = g[k]; S.red[wid][kNC + k] = nl[k]; S.red[wid][2 * kNC + k] = nr[k];
    }
    S.red[wid][3 * kNC] = dnl; S.red[wid][3 * kNC + 1] = dnr; S.okw[wid] = okm;
    S.red[wid][3 * kNC + 2] = na; S.red[wid][3 * kNC + 3] = nbb;
    S.am_v[wid] = dna; S.tq[0][wid][7] = dnb;  // (spare smem: the argmin slots are free now)
  }
  __syncthreads();

  // ---- phase 4: the tiered choice (reading 9) by thread 0
  if (tid == 0) {
    atomicMax(&A.ctr[6], (unsigned long long)(clock64() - clk_p2));
    double G[kNC], NL[kNC], NR[kNC], DNL = 0.0, DNR = 0.0, NA = 0.0, NB = 0.0, DNA = 0.0, DNB = 0.0;
    unsigned ok = (1u << kNC) - 1u;
    for (int k = 0; k < kNC; ++k) { G[k] = 0.0; NL[k] = 0.0; NR[k] = 0.0; }
    for (int w = 0; w < NW; ++w) {
      for (int k = 0; k < kNC; ++k) {
        G[k] = fmax(G[k], S.red[w][k]);
        NL[k] += S.red[w][kNC + k];
        NR[k] += S.red[w][2 * kNC + k];
      }
      DNL += S.red[w][3 * kNC]; DNR += S.red[w][3 * kNC + 1];
      NA += S.red[w][3 * kNC + 2]; NB += S.red[w][3 * kNC + 3];
      DNA += S.am_v[w]; DNB += S.tq[0][w][7];
      ok &= S.okw[w];
    }
    const double spd = P.spdiam;
    int b1 = -1, b2 = -1, b3 = -1;
    // reading 30: the interior candidate first -- taken if its child is finite
    // and its raw growth <= 8 spdiam, or <= 1e8 spdiam with the weighted
    // growth <= 64 spdiam against the four probes (the cluster's end members
    // and the two members next to the shift)
    int b_int = -1;
    if (ADJ && S.has_int && ((ok >> 6) & 1u)) {
      const double g6 = G[6];
      const double w6 = (DNL > 0 && DNR > 0 && DNA > 0 && DNB > 0)
                            ? fmax(fmax(NL[6] / DNL, NR[6] / DNR), fmax(NA / DNA, NB / DNB)) : CUDART_INF;
      if (g6 <= 8.0 * spd || (g6 <= 1e8 * spd && w6 <= A.int_wg * spd)) b_int = 6;
    }
    double r1 = 0, r2 = 0, r3 = 0;
    for (int k = 0; k < 6; ++k) {
      const bool fin = (ok >> k) & 1u;
      const double gk = fin ? G[k] : CUDART_INF;
      const double wk = (fin && DNL > 0 && DNR > 0) ? fmax(NL[k] / DNL, NR[k] / DNR) : CUDART_INF;
      if (gk <= 8.0 * spd && (b1 < 0 || gk < r1)) { b1 = k; r1 = gk; }
      if (isfinite(gk) && wk <= 64.0 * spd && (b2 < 0 || gk < r2)) { b2 = k; r2 = gk; }
      if (b3 < 0 || gk < r3) { b3 = k; r3 = gk; }
    }
    int tier = 0, best = b1;
    if (best < 0) { tier = 1; best = b2; }
    if (best < 0) { tier = 3; best = b3; if (!(r3 <= 1e8 * spd)) best = -1; }
    if (b_int >= 0) { tier = 5; best = b_int; }
    S.best = best;
    S.tier = best < 0 ? 4 : tier;
    S.sg = best < 0 ? 0.0 : S.sig[best];
    S.bad = 0;
    A.sigma_out[c] = S.sg;
    A.tier_out[c] = S.tier;
    if (best < 0) A.fail[0] = 1;
    atomicAdd(&A.ctr[0], 2ull);
  }
  __syncthreads();
  const int best = S.best;
  if (best < 0) return;

  // ---- phase 5: the chosen child, (D+_i, LLD+_i = LD_i^2 / D+_i), coalesced
  double2 *out = A.pool[c];
  bool bad = false;
#pragma unroll 4
  for (int i = tid; i < nb; i += 32 * NW) {
    const double Dp = cs_dplus(TP, QK, zs, best, i);
    const double lld = (i < nb - 1) ? __ldg(&LD[i]).y / Dp : 0.0;
    bad |= !isfinite(Dp) || Dp == 0.0 || !isfinite(lld);
    out[i] = make_double2(Dp, lld);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) A.fail[0] = 1;
}

}  // namespace mrrr
