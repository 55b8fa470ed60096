// kernels_child3.cuh -- a5: the cluster step's chains, LANE-DENSE, for the
// wide tree levels.
//
// k_child_step2 runs a cluster's ten chains (six candidate shifts, the two
// end-member probes' stationary and progressive sweeps) on the lanes of three
// warps, 11 of 96 lanes busy; at the levels with ~1000 clusters that CTA
// count made two waves of long, mostly idle warps (random n=20000: 4.7 ms per
// level).  Here a warp runs THREE clusters' chains, ten lanes each:
//   lanes 10g + 0..5   cluster g's candidate shifts (readings 8, 9),
//   lanes 10g + 6, 7   the stationary sweeps of its end-member probes,
//   lanes 10g + 8, 9   their progressive sweeps,
// every lane stepping one row per step.  The progressive step in projective
// form (a, b) -> (u = LLD b + a, a' = D a - lam u) is the stationary one with
// (D, LLD) swapped, and the backward tiles are stored reversed and swapped,
// so the forward and backward lanes run one instruction stream.  Each lane
// stages its two stored quantities per row in shared memory; at the end of a
// 16-row tile the warp writes them to the step's scratch rows with 128-byte
// stores, in k_child_step2's layout and with its arithmetic bit for bit:
//   candidates   t_i (= D+_i q_i) and q_i every 8 rows,
//   fwd probes   s_i = p_i / q_i,  rho_i = -LD_i q_i / t_i,
//   bwd probes   P_i = a_i / u_i,  sig_i = -LD_i b_{i+1} / u_{i+1}.
// k_child_step2<0, true> then runs the rest of the step (twist indices, |z|,
// growth, the tiered choice, the chosen child) on these rows.
#pragma once
#include <cuda_pipeline.h>

#include "kernels_child2.cuh"

namespace mrrr {

constexpr int kC3Lanes = 10;  // chains per cluster
constexpr int kC3Groups = 3;  // clusters per warp, at most
constexpr int kC3Warps = 1;   // warps per CTA

template <int kC3Groups>
struct C3Warp {
  double2 dl[kCRing][kC3Groups][2][kCT];  // [.][g][0]: row r0+k as (D, LLD); [.][g][1]: row r0b+15-k as (LLD, D)
  double ld[kCRing][kC3Groups][2][kCT];   // LD of the same rows
  // per lane and step (padded rows: conflict-free): A = p before the step
  // (forward probes) or after it (backward probes), B = q before, C = t
  double sa[32][kCT + 1], sb[32][kCT + 1], sc[32][kCT + 1];
};

template <int kC3Groups>
__global__ void __launch_bounds__(32 * kC3Warps) k_child_chains3(ChildArgs A) {
  __shared__ C3Warp<kC3Groups> SW[kC3Warps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  C3Warp<kC3Groups> &S = SW[wid];
  const int wbase = (blockIdx.x * kC3Warps + wid) * kC3Groups;  // the warp's first cluster (launch index)
  if (A.c0 + wbase >= A.ncl) return;  // whole warp
  const int64_t zs = A.zstride;
  const int g = min(lane / kC3Lanes, kC3Groups - 1);
  const int role = lane - kC3Lanes * g;  // 0..9; lanes beyond 10 G: >= 10 (idle)
  const bool gvalid = A.c0 + wbase + g < A.ncl;
  const bool act = gvalid && role < kC3Lanes;
  const bool bwd = role >= 8 && role < kC3Lanes;
  const bool cand = role < 6;
  // every lane keeps the three groups' rows and scratch (for the copies and
  // the stores); its own chain's shift and state
  const double2 *gDL[kC3Groups], *gLD[kC3Groups];
  double *gbase[kC3Groups];
  int gnb[kC3Groups], gnt[kC3Groups];
#pragma unroll
  for (int h = 0; h < kC3Groups; ++h) {
    gDL[h] = nullptr; gLD[h] = nullptr; gbase[h] = nullptr; gnb[h] = 0; gnt[h] = 0;
    if (A.c0 + wbase + h < A.ncl) {
      const int c = A.cl_list ? A.cl_list[A.c0 + wbase + h] : A.c0 + wbase + h;
      const Node P = A.nodes[A.cl_parent[c]];
      gDL[h] = P.DL; gLD[h] = A.LDv + P.row0; gnb[h] = P.nb; gnt[h] = (P.nb + kCT - 1) / kCT;
      gbase[h] = A.scratch + (int64_t)(wbase + h) * kCSRows * zs;
    }
  }
  int nb = 1;
  double sig = 0.0, p = 0.0, q = 1.0;
  if (gvalid) {
    const int c = A.cl_list ? A.cl_list[A.c0 + wbase + g] : A.c0 + wbase + g;
    nb = A.nodes[A.cl_parent[c]].nb;
    const int s0 = A.cl_s0[c], s1 = A.cl_s1[c] - 1;
    if (cand) {
      const double mult = (double)(1 << (role >> 1));
      if ((role & 1) == 0) {
        const double l = A.lo[s0], h = A.hi[s0];
        const double dl = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(l)), 4.0 * kEps * fabs(l));
        sig = l - mult * dl;
      } else {
        const double l = A.lo[s1], h = A.hi[s1];
        const double dr = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(h)), 4.0 * kEps * fabs(h));
        sig = h + mult * dr;
      }
    } else {
      const int side = (role - 6) & 1;  // 6, 8: left end member; 7, 9: right
      const int qs = side == 0 ? s0 : s1;
      sig = 0.5 * (A.lo[qs] + A.hi[qs]);
    }
    p = -sig; q = 1.0;
    if (bwd) {
      const double2 *DLg = A.nodes[A.cl_parent[c]].DL;
      p = __ldg(&DLg[nb - 1]).x - sig;
      if (act) A.scratch[(int64_t)(wbase + g) * kCSRows * zs + (kNC + 4 * (role - 8)) * zs + zs + nb - 1] = p;
    }
  }
  int ntmax = 0;
#pragma unroll
  for (int h = 0; h < kC3Groups; ++h) ntmax = max(ntmax, gnt[h]);
  const int ntile = (nb + kCT - 1) / kCT;
  // ring copies of tile t: per group five units of 16 copies (forward DL,
  // forward LD, backward DL swapped as two 8-byte halves, backward LD); the
  // lanes of half-warp h2 take the units u with u % 2 == h2, row lane % 16
  auto issue = [&](int t, int slot) {
    const int k = lane & (kCT - 1), h2 = lane >> 4;
#pragma unroll
    for (int u = 0; u < 5 * kC3Groups; ++u) {
      const int h = u / 5, kind = u % 5;
      const int rowf = t * kCT + k, rowb = (gnt[h] - 1 - t) * kCT + k;
      const bool on = h2 == (u & 1) && t < gnt[h] && (kind < 2 ? rowf : rowb) < gnb[h];
      const double2 *src = gDL[h] + (kind < 2 ? rowf : rowb);
      if (kind == 0) {
        if (on) __pipeline_memcpy_async(&S.dl[slot][h][0][k], src, sizeof(double2));
      } else if (kind == 1) {
        if (on) __pipeline_memcpy_async(&S.ld[slot][h][0][k], &gLD[h][rowf].x, sizeof(double));
      } else if (kind == 2) {
        if (on) __pipeline_memcpy_async(&S.dl[slot][h][1][kCT - 1 - k].x, &src->y, sizeof(double));
      } else if (kind == 3) {
        if (on) __pipeline_memcpy_async(&S.dl[slot][h][1][kCT - 1 - k].y, &src->x, sizeof(double));
      } else {
        if (on) __pipeline_memcpy_async(&S.ld[slot][h][1][kCT - 1 - k], &gLD[h][rowb].x, sizeof(double));
      }
    }
    __pipeline_commit();
  };
#pragma unroll
  for (int k = 0; k < kCRing - 1; ++k) issue(k, k);
  const int dir = bwd ? 1 : 0;
  for (int t = 0; t < ntmax; ++t) {
    __pipeline_wait_prior(kCRing - 2);
    __syncwarp();
    const int slot = t % kCRing;
    // this lane's steps in the tile: forward rows 16t + s (s < s_hi; the row
    // nb-1 without the state update); backward rows r0b + 15 - s, s >= s_lo
    // (rows r0b .. top, top <= nb - 2)
    int s_lo = 0, s_hi = 0;
    bool last = false;
    if (act && t < ntile) {
      if (!bwd) {
        s_hi = min(kCT, nb - t * kCT);
        last = t * kCT + s_hi == nb;  // the tile holds row nb-1
      } else {
        const int r0b = (ntile - 1 - t) * kCT, top = min(r0b + kCT, nb - 1) - 1;
        if (top >= r0b) { s_lo = kCT - 1 - (top - r0b); s_hi = kCT; }
      }
    }
    const double2 *TT = S.dl[slot][g][dir];
    auto step = [&](int s, bool lastrow) {
      const double2 v = TT[s];
      const double tt = fma(v.x, q, p);
      const double pn = fma(-sig, tt, v.y * p);
      S.sa[lane][s] = bwd ? pn : p;
      S.sb[lane][s] = q;
      S.sc[lane][s] = tt;
      if (!lastrow) { p = pn; q = tt; }
      if ((s & 7) == 7) {
        const double f = pow2_scale(min(max(max_exp(p, q), 1), 2045));
        p *= f; q *= f;
      }
    };
    const bool full = __all_sync(0xffffffffu, !act || (s_lo == 0 && s_hi == kCT && !last));
    if (full) {
#pragma unroll
      for (int s = 0; s < kCT; ++s) step(s, false);
    } else {
      for (int s = s_lo; s < s_hi; ++s) step(s, last && s == s_hi - 1);
    }
    __syncwarp();
    // the tile's stored quantities: chain j = 10h + r writes 16 rows of its
    // first array (lanes 0-15) and of its second (lanes 16-31), in
    // k_child_step2's layout and arithmetic
    {
      // branch-free: every lane loads and computes, only the stores are
      // predicated (a per-iteration branch compiled to reconvergence blocks)
      const int s = lane & (kCT - 1), a = lane >> 4;
      const int i_f = t * kCT + s;
      int i_b[kC3Groups];
      bool ok_b[kC3Groups], ok_f[kC3Groups];
#pragma unroll
      for (int h = 0; h < kC3Groups; ++h) {
        const int r0b = (gnt[h] - 1 - t) * kCT, top = min(r0b + kCT, gnb[h] - 1) - 1;
        i_b[h] = r0b + kCT - 1 - s;
        ok_b[h] = t < gnt[h] && i_b[h] <= top && i_b[h] >= r0b;
        ok_f[h] = t < gnt[h] && i_f < gnb[h];
      }
#pragma unroll
      for (int j = 0; j < kC3Groups * kC3Lanes; ++j) {
        const int h = j / kC3Lanes, r = j % kC3Lanes;
        double *bs = gbase[h];
        if (r < 6) {
          // t_i (lanes 0-15), q_i at rows i % 8 == 0 (lanes 16, 24)
          const double val = a == 0 ? S.sc[j][s] : S.sb[j][s];
          double *dst = a == 0 ? bs + r * zs + i_f : bs + (kNC + 10) * zs + r * (zs / 8) + (i_f >> 3);
          if (ok_f[h] && (a == 0 || (s & 7) == 0)) *dst = val;
        } else {
          // first array: s_i = A / B (forward) or P_i = A / C (backward);
          // second: rho_i / sig_i = -LD_i * (B / C)
          const bool b8 = r >= 8;
          const double ldv = S.ld[slot][h][b8 ? 1 : 0][s];
          const double A_ = S.sa[j][s], B_ = S.sb[j][s], C_ = S.sc[j][s];
          const double num = a == 0 ? A_ : B_, den = (a == 0 && !b8) ? B_ : C_;
          const double d = div_nr(num, den);
          const double val = a == 0 ? d : -ldv * d;
          double *pr = bs + (kNC + 4 * ((r - 6) & 1)) * zs;
          if (!b8) {
            double *dst = pr + (a == 0 ? 0 : 2) * zs + i_f;
            if (ok_f[h] && (a == 0 || i_f < gnb[h] - 1)) *dst = val;
          } else {
            double *dst = pr + (a == 0 ? 1 : 3) * zs + i_b[h];
            if (ok_b[h]) *dst = val;
          }
        }
      }
    }
    __syncwarp();
    issue(t + kCRing - 1, (t + kCRing - 1) % kCRing);
  }
  __pipeline_wait_prior(0);
}

}  // namespace mrrr
