// kernels_probe.cuh -- a5 probes: the parent's eigenvector at each end
// eigenvalue of a cluster, which only weights the tier-(ii) growth test of the
// child shift (reading 9, §4.5).  One CTA of two warps per probe.
//
// The twisted factorization of L D L^T - lambda I is
// two independent recurrences: the stationary one from the top and the
// progressive one from the bottom.  Warp 0 runs the first and warp 1 the
// second AT THE SAME TIME (the two dependent chains overlap instead of
// following each other), each storing per row the ratios the rest needs:
//   forward,  state (p_i, q_i) before row i:  s_i = p_i / q_i,
//             rho_i = z_i / z_{i+1} = -LD_i q_i / t_i          (i < nb - 1)
//   backward, state (a_i, b_i) at row i:      P_i = a_i / b_i,
//             sig_i = z_{i+1} / z_i = -LD_i b_{i+1} / u_{i+1}  (i < nb - 1)
// Then all 64 threads find r = argmin |gamma_i|, gamma_i = s_i + P_i + lambda
// (ties to the lower row), and form z with z_r = 1 by a scan of log2 |ratio|
// in both directions: z_i = 2^(sum of log2 |rho_k|, k = i..r-1) above r,
// 2^(sum of log2 |sig_k|, k = r..i-1) below.  Only z_i^2 is used downstream
// (sum |D+_i| z_i^2 / sum z_i^2), so |z_i| is stored.  Every lane of a chain
// warp runs the same chain (no divergence); lane k keeps row k's values of a
// 16-row tile, divides once per tile and stores them with one coalesced
// write.  Rows come through a cp.async ring as in kernels_child.cuh.
#pragma once
#include <cuda_pipeline.h>

#include "common.cuh"
#include "kernels_vec.cuh"

namespace mrrr {

constexpr int kPT = 16;    // rows per tile
constexpr int kPRing = 6;  // tiles in flight

struct ProbeSmem {
  double2 rDL[2][kPRing][kPT];  // per chain warp: (D, LLD)
  double2 rLD[2][kPRing][kPT];  //                (LD, LD^2)
  double red_v[2];
  int red_i[2];
};

struct ProbeArgs {
  const Node *nodes;
  const VecTask *tasks;     // probe t: node, slot (end member), col = output vector index
  int ntask;
  const double2 *LDv;       // global (LD, LD^2) per row
  const double *lo, *hi;    // slot brackets (node coordinates)
  double *zbuf;             // |z| of probe t at zbuf + col * zstride
  int64_t zstride;
  double *scratch;          // 4 * zstride doubles per probe: s, P, rho, sig
  unsigned long long *ctr;  // [0] factorizations
};

__global__ void __launch_bounds__(64) k_probe(ProbeArgs A) {
  __shared__ ProbeSmem S;
  const int t = blockIdx.x;
  if (t >= A.ntask) return;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const VecTask tk = A.tasks[t];
  const Node N = A.nodes[tk.node];
  const int nb = N.nb;
  double *z = A.zbuf + tk.col * A.zstride;
  if (nb == 1) {
    if (threadIdx.x == 0) { z[0] = 1.0; atomicAdd(&A.ctr[0], 1ull); }
    return;
  }
  const double lam = 0.5 * (A.lo[tk.slot] + A.hi[tk.slot]);
  double *sS = A.scratch + (int64_t)t * 4 * A.zstride;
  double *sP = sS + A.zstride, *sR = sP + A.zstride, *sG = sR + A.zstride;
  const double2 *DL = N.DL, *LD = A.LDv + N.row0;
  const int ntile = (nb + kPT - 1) / kPT;

  // ---- phase 1: the two chains, one per warp
  {
    const bool up = wid == 0;
    auto tile_of = [&](int c) { return up ? c : ntile - 1 - c; };  // c-th tile visited
    auto issue = [&](int c) {
      const int slot = c % kPRing;
      const int k = lane & (kPT - 1);
      if (c < ntile) {
        const int row = tile_of(c) * kPT + k;
        if (row < nb) {
          if (lane < kPT) __pipeline_memcpy_async(&S.rDL[wid][slot][k], &DL[row], sizeof(double2));
          else __pipeline_memcpy_async(&S.rLD[wid][slot][k], &LD[row], sizeof(double2));
        }
      }
      __pipeline_commit();
    };
#pragma unroll
    for (int k = 0; k < kPRing - 1; ++k) issue(k);
    if (up) {
      double p = -lam, q = 1.0;
      for (int c = 0; c < ntile; ++c) {
        __pipeline_wait_prior(kPRing - 2);
        __syncwarp();
        const int slot = c % kPRing, r0 = c * kPT, rows = min(kPT, nb - r0);
        double kp = 0.0, kq = 1.0, kt = 1.0, kld = 0.0;
        auto row = [&](int k) {
          const int i = r0 + k;
          const double2 v = S.rDL[0][slot][k];
          const double ld = S.rLD[0][slot][k].x;
          const double tt = fma(v.x, q, p);
          if (lane == k) { kp = p; kq = q; kt = tt; kld = ld; }
          if (i < nb - 1) { p = fma(-lam, tt, v.y * p); q = tt; }
          if ((k & 7) == 7) {
            const double f = pow2_scale(min(max(max_exp(p, q), 1), 2045));
            p *= f; q *= f;
          }
        };
        if (rows == kPT) {
#pragma unroll
          for (int k = 0; k < kPT; ++k) row(k);
        } else {
          for (int k = 0; k < rows; ++k) row(k);
        }
        if (lane < rows) {
          const int i = r0 + lane;
          sS[i] = kp / kq;
          if (i < nb - 1) sR[i] = -kld * (kq / kt);
        }
        __syncwarp();
        issue(c + kPRing - 1);
      }
    } else {
      double a = __ldg(&DL[nb - 1]).x - lam, b = 1.0;
      if (lane == 0) sP[nb - 1] = a;
      for (int c = 0; c < ntile; ++c) {
        __pipeline_wait_prior(kPRing - 2);
        __syncwarp();
        const int slot = c % kPRing, r0 = tile_of(c) * kPT;
        const int top = min(r0 + kPT, nb - 1) - 1;  // rows r0 .. top step (row i from i+1)
        double kb = 1.0, ku = 1.0, ka = 0.0, kld = 0.0;
        auto row = [&](int k) {
          const double2 v = S.rDL[1][slot][k];
          const double ld = S.rLD[1][slot][k].x;
          const double u = fma(v.y, b, a);
          const double an = fma(-lam, u, v.x * a);
          if (lane == k) { kb = b; ku = u; ka = an; kld = ld; }
          a = an; b = u;
          if ((k & 7) == 0) {
            const double f = pow2_scale(min(max(max_exp(a, b), 1), 2045));
            a *= f; b *= f;
          }
        };
        if (top - r0 + 1 == kPT) {
#pragma unroll
          for (int k = kPT - 1; k >= 0; --k) row(k);
        } else {
          for (int k = top - r0; k >= 0; --k) row(k);
        }
        if (lane <= top - r0) {
          const int i = r0 + lane;
          sP[i] = ka / ku;
          sG[i] = -kld * (kb / ku);
        }
        __syncwarp();
        issue(c + kPRing - 1);
      }
    }
    __pipeline_wait_prior(0);
  }
  __syncthreads();

  // ---- phase 2: r = argmin |gamma_i| (ties to the lower row)
  double bv = CUDART_INF;
  int bi = nb;
  for (int i = threadIdx.x; i < nb; i += 64) {
    const double g = fabs(sS[i] + sP[i] + lam);
    if (g < bv) { bv = g; bi = i; }  // ascending i per thread: first minimum kept
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) { S.red_v[wid] = bv; S.red_i[wid] = bi; }
  __syncthreads();
  int r;
  {
    const double v0 = S.red_v[0], v1 = S.red_v[1];
    const int i0 = S.red_i[0], i1 = S.red_i[1];
    r = (v1 < v0 || (v1 == v0 && i1 < i0)) ? i1 : i0;
    if (r >= nb) r = nb - 1;  // no finite gamma: any twist (weights only)
  }

  // ---- phase 3: |z| by log2 scans, warp 0 upward from r (rows r-1 .. 0),
  // warp 1 downward (rows r+1 .. nb-1)
  if (wid == 0) {
    if (lane == 0) z[r] = 1.0;
    double carry = 0.0;  // log2 |z_{i+1}| for the tile's first row (from r)
    for (int top = r - 1; top >= 0; top -= 32) {
      const int i = top - lane;  // lane 0 nearest r
      double l = 0.0;
      if (i >= 0) l = fmin(fmax(log2(fabs(sR[i])), -4096.0), 4096.0);
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, l, o);
        if (lane >= o) l += y;
      }
      const double L = carry + l;
      if (i >= 0) z[i] = exp2(L);
      carry = __shfl_sync(0xffffffffu, L, 31);
    }
  } else {
    double carry = 0.0;
    for (int bot = r; bot < nb - 1; bot += 32) {
      const int i = bot + lane;  // z_{i+1} from sig_i
      double l = 0.0;
      if (i < nb - 1) l = fmin(fmax(log2(fabs(sG[i])), -4096.0), 4096.0);
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, l, o);
        if (lane >= o) l += y;
      }
      const double L = carry + l;
      if (i < nb - 1) z[i + 1] = exp2(L);
      carry = __shfl_sync(0xffffffffu, L, 31);
    }
  }
  if (threadIdx.x == 0) atomicAdd(&A.ctr[0], 1ull);
}

}  // namespace mrrr
