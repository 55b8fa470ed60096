// kernels_child.cuh -- a5: the cluster step of one tree level in one kernel
// (SURVEY §8(c) O9), one warp per cluster.
//
// Pass 1: lanes 0..5 run the six candidate shifts (offsets 1, 2, 4 beyond
// each cluster end, readings 8 and 9) through the projective
// stationary transform of the parent, accumulating the raw growth max|D+|
// and the growth weighted by the parent's two end-eigenvalue vectors (the
// probes of k_wprobe).  The tiered choice is made in-warp.  Pass 2: every
// lane runs the chosen shift's transform (the same instruction stream), the
// chain values of each 16-row tile go to shared memory and lane k forms row
// k's (D+_k, LLD+_k = LD_k^2 / D+_k), stored with one coalesced 256-byte
// write per tile.  Rows come through a shared-memory ring filled by cp.async
// ahead of the chains (as in kernels_warp.cuh).  Replaces k_cand + k_pick +
// k_child_chain + k_child_finish (same arithmetic as those).
#pragma once
#include <cuda_pipeline.h>

#include "common.cuh"

namespace mrrr {

constexpr int kCT = 16;         // rows per tile
constexpr int kCRing = 6;       // tiles in flight
constexpr int kCWarps = 4;      // warps (clusters) per CTA

struct ChildSmem {
  double2 rDL[kCRing][kCT];     // parent (D, LLD)
  double rZL[kCRing][kCT], rZR[kCRing][kCT];  // probe vectors (pass 1)
  double2 rLD[kCRing][kCT];     // block (LD, LD^2) (pass 2)
  double tq[2][kCT];            // pass 2: t_i and q_i of the tile
};

struct ChildArgs {
  const Node *nodes;
  const int *cl_parent, *cl_s0, *cl_s1;
  const double *lo, *hi;
  const double *zbuf;           // probes: rows of cluster c at zbuf + (2c + side) * zstride
  int64_t zstride;
  const double2 *LDv;           // global (LD, LD^2) per row
  int ncl;
  double rtol;
  double2 *pool;                // child c's rows at pool + c * stride
  int64_t stride;
  double *sigma_out;
  int *tier_out;
  int *fail;
};

__global__ void __launch_bounds__(32 * kCWarps) k_child_warp(ChildArgs A) {
  __shared__ ChildSmem smem[kCWarps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kCWarps + wid;
  if (c >= A.ncl) return;
  ChildSmem &S = smem[wid];
  const Node P = A.nodes[A.cl_parent[c]];
  const int nb = P.nb;
  const int s0 = A.cl_s0[c], s1 = A.cl_s1[c] - 1;
  const double *zl = A.zbuf + (int64_t)(2 * c) * A.zstride;
  const double *zr = A.zbuf + (int64_t)(2 * c + 1) * A.zstride;
  const double2 *LDb = A.LDv + P.row0;
  const int ntile = (nb + kCT - 1) / kCT;

  // ---- candidate shift of this lane (lanes >= 6 duplicate lane 0)
  const int which = lane < 6 ? lane : 0;
  const double mult = (double)(1 << (which >> 1));
  double sigma;
  if ((which & 1) == 0) {
    const double l = A.lo[s0], h = A.hi[s0];
    const double dl = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(l)), 4.0 * kEps * fabs(l));
    sigma = l - mult * dl;
  } else {
    const double l = A.lo[s1], h = A.hi[s1];
    const double dr = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(h)), 4.0 * kEps * fabs(h));
    sigma = h + mult * dr;
  }

  // ---- pass 1: growth of the six candidates
  auto issue1 = [&](int t) {
    const int slot = t % kCRing;
    const int k = lane & (kCT - 1), row = t * kCT + k;
    if (t < ntile && row < nb) {
      if (lane < kCT) __pipeline_memcpy_async(&S.rDL[slot][k], &P.DL[row], sizeof(double2));
      else {
        __pipeline_memcpy_async(&S.rZL[slot][k], &zl[row], sizeof(double));
        __pipeline_memcpy_async(&S.rZR[slot][k], &zr[row], sizeof(double));
      }
    }
    __pipeline_commit();
  };
  double p = -sigma, q = 1.0, g = 0.0, nl = 0.0, dnl = 0.0, nr = 0.0, dnr = 0.0;
  bool fin = true;
#pragma unroll
  for (int k = 0; k < kCRing - 1; ++k) issue1(k);
  for (int t = 0; t < ntile; ++t) {
    __pipeline_wait_prior(kCRing - 2);
    __syncwarp();
    const int slot = t % kCRing, r0 = t * kCT;
    const int rows = min(kCT, nb - r0);
    auto row = [&](int k) {
      const int i = r0 + k;
      const double2 v = S.rDL[slot][k];
      const double a = S.rZL[slot][k], b = S.rZR[slot][k];
      const double tt = fma(v.x, q, p);
      const double dp = tt * rcp_nr(q);  // D+_i (off the recurrence chain, branch-free)
      fin &= isfinite(dp) && dp != 0.0;
      const double adp = fabs(dp);
      g = fmax(g, adp);
      nl = fma(adp, a * a, nl); dnl = fma(a, a, dnl);
      nr = fma(adp, b * b, nr); dnr = fma(b, b, dnr);
      if (i < nb - 1) { p = fma(-sigma, tt, v.y * p); q = tt; }
      if ((k & 7) == 7) {
        const int ee = max_exp(p, q);
        fin &= ee < 2047;
        const double f = pow2_scale(min(ee, 2045));
        p *= f; q *= f;
      }
    };
    if (rows == kCT) {
#pragma unroll
      for (int k = 0; k < kCT; ++k) row(k);
    } else {
      for (int k = 0; k < rows; ++k) row(k);
    }
    __syncwarp();
    issue1(t + kCRing - 1);
  }
  __pipeline_wait_prior(0);
  const double raw = fin ? g : CUDART_INF;
  const double wgt = (fin && dnl > 0 && dnr > 0) ? fmax(nl / dnl, nr / dnr) : CUDART_INF;

  // ---- tiered choice (reading 9, as k_pick)
  const double spd = P.spdiam;
  int b1 = -1, b2 = -1, b3 = -1;
  double r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double gk = __shfl_sync(0xffffffffu, raw, k);
    const double wk = __shfl_sync(0xffffffffu, wgt, k);
    if (gk <= 8.0 * spd && (b1 < 0 || gk < r1)) { b1 = k; r1 = gk; }
    if (isfinite(gk) && wk <= 64.0 * spd && (b2 < 0 || gk < r2)) { b2 = k; r2 = gk; }
    if (b3 < 0 || gk < r3) { b3 = k; r3 = gk; }
  }
  int tier = 0, best = b1;
  if (best < 0) { tier = 1; best = b2; }
  if (best < 0) { tier = 3; best = b3; if (!(r3 <= 1e8 * spd)) best = -1; }
  if (best < 0) {
    if (lane == 0) { A.sigma_out[c] = 0.0; A.tier_out[c] = 4; A.fail[0] = 1; }
    return;
  }
  const double sg = __shfl_sync(0xffffffffu, sigma, best);
  if (lane == 0) { A.sigma_out[c] = sg; A.tier_out[c] = tier; }

  // ---- pass 2: the chosen child, (D+_i, LLD+_i = LD_i^2 / D+_i)
  double2 *out = A.pool + (int64_t)c * A.stride;
  auto issue2 = [&](int t) {
    const int slot = t % kCRing;
    const int k = lane & (kCT - 1), row = t * kCT + k;
    if (t < ntile && row < nb) {
      if (lane < kCT) __pipeline_memcpy_async(&S.rDL[slot][k], &P.DL[row], sizeof(double2));
      else __pipeline_memcpy_async(&S.rLD[slot][k], &LDb[row], sizeof(double2));
    }
    __pipeline_commit();
  };
  p = -sg; q = 1.0;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kCRing - 1; ++k) issue2(k);
  for (int t = 0; t < ntile; ++t) {
    __pipeline_wait_prior(kCRing - 2);
    __syncwarp();
    const int slot = t % kCRing, r0 = t * kCT;
    const int rows = min(kCT, nb - r0);
    auto row = [&](int k) {
      const int i = r0 + k;
      const double2 v = S.rDL[slot][k];
      const double tt = fma(v.x, q, p);
      if (lane == 0) { S.tq[0][k] = tt; S.tq[1][k] = q; }
      if (i < nb - 1) { p = fma(-sg, tt, v.y * p); q = tt; }
      if ((k & 7) == 7) {
        const int ee = max_exp(p, q);
        const double f = pow2_scale(min(max(ee, 1), 2045));
        p *= f; q *= f;
      }
    };
    if (rows == kCT) {
#pragma unroll
      for (int k = 0; k < kCT; ++k) row(k);
    } else {
      for (int k = 0; k < rows; ++k) row(k);
    }
    __syncwarp();
    if (lane < rows) {
      const int i = r0 + lane;
      const double Dp = S.tq[0][lane] / S.tq[1][lane];
      const double ld2 = (i < nb - 1) ? S.rLD[slot][lane].y : 0.0;
      const double lld = (i < nb - 1) ? ld2 / Dp : 0.0;
      bad |= !isfinite(Dp) || Dp == 0.0 || !isfinite(lld);
      out[i] = make_double2(Dp, lld);
    }
    __syncwarp();
    issue2(t + kCRing - 1);
  }
  __pipeline_wait_prior(0);
  if (__any_sync(0xffffffffu, bad) && lane == 0) A.fail[0] = 1;
}

}  // namespace mrrr
