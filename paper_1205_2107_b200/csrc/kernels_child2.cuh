// kernels_child2.cuh -- a5: the cluster step with the chains PACKED into the
// lanes of two warps.
//
// The same arithmetic as k_child_step (kernels_child.cuh), bit for bit, on a
// CTA of three warps instead of five (nine): k_child_step runs every dependent
// chain on a whole warp (32 lanes computing the same chain, lane k keeping
// row k's values for the coalesced stores), so at the wide tree levels --
// ~1000 clusters, issue-bound -- it spent ~32 warp-instructions per useful
// chain step.  Here every chain is one LANE:
//   warp 0 (top-down over the parent's rows): lanes 0..6 the seven candidate
//          shifts (readings 8, 9, 30);
//   warp 1 (top-down): lanes 0, 1 the stationary sweeps of the end-member
//          probes, lanes 2, 3 (ADJ) those of the probes next to the interior
//          shift;
//   warp 2 (bottom-up): lanes 0, 1 (2, 3 with ADJ) the progressive sweeps of
//          the same probes.
// (The candidates and the forward probes share the row order but not the
// per-tile work -- stores for the former, two divisions per row for the
// latter -- so they run on two warps: one warp for both made the level-0
// step, which is latency-bound, 30 % slower.)
// All chain lanes of a warp read the same parent row at each step (a
// broadcast from the cp.async ring), stage their per-row values (p, q, t) in
// shared memory, and at the end of each 16-row tile the warp's 32 lanes turn
// the staged values into the stored quantities -- t and q for the
// candidates, s = p/q and rho = -LD q/t for the probes (P = a/u and
// sig = -LD b/u backward) -- with the divisions spread over the lanes and
// the stores coalesced.  The later phases (twist index and |z| per probe,
// growth, tiered choice, the chosen child) are k_child_step's, on 64 threads.
#pragma once
#include <cuda_pipeline.h>

#include "kernels_child.cuh"

namespace mrrr {

constexpr int kCF = 11;  // chain lanes of warp F: 7 candidates + 4 probes
constexpr int kCB = 4;   // chain lanes of warp B: 4 probes

struct Child2Smem {
  ChainRing ring[3];
  double stF[kCT][kCF][3];  // warp F staging: (p, q, t) per row and chain lane
  double stB[kCT][kCB][3];  // warp B staging: (b, u, a) per row and chain lane
  double red[4][3 * kNC + 4];
  unsigned okw[4];
  double am2[4][2];         // per warp: the denominators of the ADJ weights
  double sig[kNC];
  int has_int, jint;
  double sig_int;
  double gbw[3];
  int gjw[3];
  int best, tier;
  double sg;
  int rr[2];  // POST: the probes' twist indices
};

// POST = true (ADJ = 0): the chains were run by k_child_chains3
// (kernels_child3.cuh), which wrote the same scratch rows; phase 1 only sets
// the candidates' shifts.
template <int ADJ, bool POST = false>
// resident CTAs per SM asked of ptxas for k_child_step2<0>: 6 (96 registers,
// 284 B of spills) against 4 (168 registers, none).  Measured on B200 with
// the vector pieces overlapping (bench, 20 steps, twice each): random n=20000
// 51.3 -> 49.0 ms, n=1e5 1084 -> 1073 ms; alone (MRRR_TRACE=2) the wide
// levels' steps get slower (4.07 -> 4.71 ms), so the gain is in sharing the
// SMs with the vector warps.  5 (128 registers): 54.3 ms; 8 (80): 49.4 ms.
#ifndef MRRR_CS2_MINB
#define MRRR_CS2_MINB 6
#endif
#ifndef MRRR_CS2P_MINB
#define MRRR_CS2P_MINB 6
#endif
__global__ void __launch_bounds__(POST ? 128 : 96, ADJ ? 2 : POST ? MRRR_CS2P_MINB : MRRR_CS2_MINB) k_child_step2(ChildArgs A) {
  constexpr int NPROBE = 2 + 2 * ADJ;  // probe sides
  __shared__ Child2Smem S;
  if (A.c0 + (int)blockIdx.x >= A.ncl) return;
  const int c = A.cl_list ? A.cl_list[A.c0 + blockIdx.x] : A.c0 + (int)blockIdx.x;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const Node P = A.nodes[A.cl_parent[c]];
  const int nb = P.nb;
  const int s0 = A.cl_s0[c], s1 = A.cl_s1[c] - 1;
  const double2 *DL = P.DL, *LD = A.LDv + P.row0;
  const int64_t zs = A.zstride;
  constexpr int ROWS = ADJ ? kCSRowsAdj : kCSRows;
  double *base = A.scratch + (int64_t)blockIdx.x * ROWS * zs;
  double *TP = base;
  double *QK = base + (kNC + 10) * zs;
  double *pr[4] = {base + kNC * zs, base + (kNC + 4) * zs, base + kCSRows * zs, base + (kCSRows + 4) * zs};
  double *zz[4] = {base + (kNC + 8) * zs, base + (kNC + 9) * zs, base + (kCSRows + 8) * zs, base + (kCSRows + 9) * zs};

  // ---- phase 0 (ADJ): the interior candidate (reading 30), as in k_child_step
  if (ADJ) {
    const int mm = s1 - s0 + 1;
    double gb = -CUDART_INF;
    int jbest = -1;
    if (A.shift_strategy == 1 && mm >= 2000 && A.hi[s1] - A.lo[s0] > 1e-6 * P.spdiam) {
      const int ja = s0 + mm / 4, jb = s1 - mm / 4;
      for (int j = ja + tid; j < jb; j += 96) {
        const double gj = A.lo[j + 1] - A.hi[j];
        if (gj > gb) { gb = gj; jbest = j; }
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, gb, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jbest, o);
      if (og > gb || (og == gb && oj >= 0 && (jbest < 0 || oj < jbest))) { gb = og; jbest = oj; }
    }
    if (lane == 0) { S.gbw[wid] = gb; S.gjw[wid] = jbest; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < 3; ++w) {
        const double og = S.gbw[w];
        const int oj = S.gjw[w];
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
  const bool has_int = ADJ && S.has_int;
  auto probe_slot = [&](int side) { return side == 0 ? s0 : side == 1 ? s1 : S.jint + (side - 2); };
  auto probe_lam = [&](int side) {
    const int q = probe_slot(side);
    return 0.5 * (A.lo[q] + A.hi[q]);
  };

  // ---- phase 1: the chains, one per lane
  const long long clk_p0 = clock64();
  const int ntile = (nb + kCT - 1) / kCT;
  ChainRing &R = S.ring[wid];
  if (POST) {
    if (tid < 6) {
      const int which = tid;
      const double mult = (double)(1 << (which >> 1));
      if ((which & 1) == 0) {
        const double l = A.lo[s0], h = A.hi[s0];
        const double dl = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(l)), 4.0 * kEps * fabs(l));
        S.sig[tid] = l - mult * dl;
      } else {
        const double l = A.lo[s1], h = A.hi[s1];
        const double dr = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(h)), 4.0 * kEps * fabs(h));
        S.sig[tid] = h + mult * dr;
      }
    }
  } else if (wid < 2) {
    // warps 0, 1: this lane's chain: a candidate (warp 0) or a forward probe (warp 1)
    const int cb = wid == 0 ? 0 : kNC, nf = wid == 0 ? kNC : NPROBE;
    const int ch = cb + (lane < nf ? lane : 0);
    double sigma;
    if (ch < kNC) {
      const int which = ch < 6 ? ch : 0;
      const double mult = (double)(1 << (which >> 1));
      if (ch == 6 && has_int) {
        sigma = S.sig_int;
      } else if ((which & 1) == 0) {
        const double l = A.lo[s0], h = A.hi[s0];
        const double dl = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(l)), 4.0 * kEps * fabs(l));
        sigma = l - mult * dl;
      } else {
        const double l = A.lo[s1], h = A.hi[s1];
        const double dr = fmax(fmax(2.0 * (h - l), 2.0 * A.rtol * fabs(h)), 4.0 * kEps * fabs(h));
        sigma = h + mult * dr;
      }
    } else {
      sigma = probe_lam(ch - kNC);  // the probe's lambda: the same recurrence with mu = lambda
    }
    if (wid == 0 && lane < kNC) S.sig[lane] = sigma;
#pragma unroll
    for (int k = 0; k < kCRing - 1; ++k) cs_issue(R, DL, LD, nb, k < ntile ? k : -1, k, lane, true);
    double p = -sigma, q = 1.0;
    for (int t = 0; t < ntile; ++t) {
      __pipeline_wait_prior(kCRing - 2);
      __syncwarp();
      const int slot = t % kCRing, r0 = t * kCT, rows = min(kCT, nb - r0);
      auto row = [&](const double2 v, int k, bool last_check) {
        const int i = r0 + k;
        const double tt = fma(v.x, q, p);
        if (lane < nf) { S.stF[k][cb + lane][0] = p; S.stF[k][cb + lane][1] = q; S.stF[k][cb + lane][2] = tt; }
        if (!last_check || i < nb - 1) { p = fma(-sigma, tt, v.y * p); q = tt; }
        if ((k & 7) == 7) {
          const double f = pow2_scale(min(max(max_exp(p, q), 1), 2045));
          p *= f; q *= f;
        }
      };
      if (rows == kCT && r0 + kCT < nb) {
#pragma unroll
        for (int h = 0; h < kCT; h += 8) {
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
      // the tile's stored quantities, spread over the warp (k_child_step's
      // values: t, q every 8 rows; s = p/q, rho = -LD q/t)
      for (int e = lane; e < nf * kCT; e += 32) {
        const int cc = cb + e / kCT, k = e % kCT, i = r0 + k;
        if (k >= rows) continue;
        const double sp = S.stF[k][cc][0], sq = S.stF[k][cc][1], st = S.stF[k][cc][2];
        if (cc < kNC) {
          TP[cc * zs + i] = st;
          if ((k & 7) == 0) QK[cc * (zs / 8) + (i >> 3)] = sq;
        } else {
          double *qq = pr[cc - kNC];
          qq[i] = div_nr(sp, sq);
          if (i < nb - 1) qq[2 * zs + i] = -R.rLD[slot][k].x * div_nr(sq, st);
        }
      }
      __syncwarp();
      const int cn = t + kCRing - 1;
      cs_issue(R, DL, LD, nb, cn < ntile ? cn : -1, cn % kCRing, lane, true);
    }
    __pipeline_wait_prior(0);
  } else {
    // warp B: the progressive sweeps of the probes
    const int side = lane < NPROBE ? lane : 0;
    const double lam = probe_lam(side);
#pragma unroll
    for (int k = 0; k < kCRing - 1; ++k) cs_issue(R, DL, LD, nb, k < ntile ? ntile - 1 - k : -1, k, lane, true);
    double a = __ldg(&DL[nb - 1]).x - lam, b = 1.0;
    if (lane < NPROBE && (lane < 2 || has_int)) pr[side][zs + nb - 1] = a;
    for (int t = 0; t < ntile; ++t) {
      __pipeline_wait_prior(kCRing - 2);
      __syncwarp();
      const int slot = t % kCRing, r0 = (ntile - 1 - t) * kCT;
      const int top = min(r0 + kCT, nb - 1) - 1;  // rows r0 .. top step (row i from i+1)
      auto row = [&](const double2 v, int k) {
        const double u = fma(v.y, b, a);
        const double an = fma(-lam, u, v.x * a);
        if (lane < NPROBE) { S.stB[k][lane][0] = b; S.stB[k][lane][1] = u; S.stB[k][lane][2] = an; }
        a = an; b = u;
        if ((k & 7) == 0) {
          const double f = pow2_scale(min(max(max_exp(a, b), 1), 2045));
          a *= f; b *= f;
        }
      };
      if (top - r0 + 1 == kCT) {
#pragma unroll
        for (int h = kCT - 8; h >= 0; h -= 8) {
          double2 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = R.rDL[slot][h + k];
#pragma unroll
          for (int k = 7; k >= 0; --k) row(v[k], h + k);
        }
      } else {
        for (int k = top - r0; k >= 0; --k) row(R.rDL[slot][k], k);
      }
      __syncwarp();
      for (int e = lane; e < NPROBE * kCT; e += 32) {
        const int cc = e / kCT, k = e - cc * kCT, i = r0 + k;
        if (k > top - r0) continue;
        const double sb = S.stB[k][cc][0], su = S.stB[k][cc][1], sa = S.stB[k][cc][2];
        double *qq = pr[cc];
        qq[zs + i] = div_nr(sa, su);                           // P_i
        qq[3 * zs + i] = -R.rLD[slot][k].x * div_nr(sb, su);   // sig_i
      }
      __syncwarp();
      const int cn = t + kCRing - 1;
      cs_issue(R, DL, LD, nb, cn < ntile ? ntile - 1 - cn : -1, cn % kCRing, lane, true);
    }
    __pipeline_wait_prior(0);
  }
  if (!POST && lane == 0) atomicMax(&A.ctr[1 + (wid == 0 ? 1 : wid == 1 ? 3 : 2)], (unsigned long long)(clock64() - clk_p0));
  __syncthreads();
  const long long clk_p1 = clock64();

  // ---- phase 2: each probe's twist index and |z| (the up and down scans
  // from r).  Without POST warp w takes the sides w, w + 3, each side's
  // argmin and two scans in sequence; with POST (four warps, ADJ = 0) the two
  // argmins run on warps 0, 1 and then the four scans on one warp each --
  // the same per-side arithmetic, so the same values
  constexpr double kDead = -1.0e9;
  auto split = [](double x, double &mm, double &ee) {
    const long long bb = __double_as_longlong(x) & 0x7fffffffffffffffLL;
    const int ex = (int)(bb >> 52);
    const bool ok = ex > 0 && ex < 2047;
    mm = ok ? __longlong_as_double((bb & 0x000fffffffffffffLL) | 0x3ff0000000000000LL) : 1.0;
    ee = ok ? (double)(ex - 1023) : kDead;
  };
  auto mul = [](double &mm, double &ee, double m2, double e2) {
    mm *= m2; ee += e2;
    if (mm >= 2.0) { mm *= 0.5; ee += 1.0; }
  };
  auto to_double = [](double mm, double ee) {
    if (ee < -1022.0) return 0.0;
    if (ee > 1023.0) return CUDART_INF;
    const int ei = (int)ee;
    return __hiloint2double(__double2hiint(mm) + (ei << 20), __double2loint(mm));
  };
  auto twist_of = [&](int side) {  // r = argmin |s_i + P_i + lam| (ties: lowest i), z[r] = 1
    const double lam = probe_lam(side);
    const double *sS = pr[side], *sP = pr[side] + zs;
    double bv = CUDART_INF;
    int bi = nb;
#pragma unroll 8
    for (int i = lane; i < nb; i += 32) {
      const double g = fabs(sS[i] + sP[i] + lam);
      if (g < bv) { bv = g; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    int r = bi;
    if (r >= nb) r = nb - 1;
    if (lane == 0) zz[side][r] = 1.0;
    return r;
  };
  auto scan_from = [&](int side, int dirn, int r) {  // |z| of the rows above (dirn 0) or below (1) r
    const double *sR = pr[side] + 2 * zs, *sG = pr[side] + 3 * zs;
    double *z = zz[side];
    const bool up = dirn == 0;
    const int m = up ? r : nb - 1 - r;
    const double *src = up ? sR + (r - 1) : sG + r;
    const int dir = up ? -1 : 1;
    double *dst = up ? z + (r - 1) : z + (r + 1);
    double cm = 1.0, ce = 0.0;
    constexpr int kBlk = 8;
    for (int b0 = 0; b0 < m; b0 += 32 * kBlk) {
      double xv[kBlk];
#pragma unroll
      for (int u = 0; u < kBlk; ++u) {
        const int j = b0 + u * 32 + lane;
        xv[u] = j < m ? src[dir * j] : 1.0;
      }
#pragma unroll
      for (int u = 0; u < kBlk; ++u) {
        const int j = b0 + u * 32 + lane;
        double im, ie;
        split(xv[u], im, ie);
        if (j >= m) { im = 1.0; ie = 0.0; }
        for (int o = 1; o < 32; o <<= 1) {
          const double ym = __shfl_up_sync(0xffffffffu, im, o), ye = __shfl_up_sync(0xffffffffu, ie, o);
          if (lane >= o) mul(im, ie, ym, ye);
        }
        mul(im, ie, cm, ce);
        if (j < m) dst[dir * j] = to_double(im, ie);
        cm = __shfl_sync(0xffffffffu, im, 31);
        ce = __shfl_sync(0xffffffffu, ie, 31);
      }
    }
  };
  // POST's scan: each lane multiplies 8 consecutive ratios serially, one
  // warp scan combines the 32 lane products (5 shuffle steps per 256 rows
  // instead of 40), and each lane applies its prefix to its 8 values.  The
  // same (mantissa, exponent) products in another association order: |z| may
  // differ from k_child_step2's in the last bits (a weight of the growth
  // test, reading 27; GPU test test_schedule_invariance compares the
  // solves)
  auto scan_from_lanes = [&](int side, int dirn, int r) {
    const double *sR = pr[side] + 2 * zs, *sG = pr[side] + 3 * zs;
    double *z = zz[side];
    const bool up = dirn == 0;
    const int m = up ? r : nb - 1 - r;
    const double *src = up ? sR + (r - 1) : sG + r;
    const int dir = up ? -1 : 1;
    double *dst = up ? z + (r - 1) : z + (r + 1);
    constexpr int kL = 8;
    double cm = 1.0, ce = 0.0;
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
      // inclusive scan of the lane products, then the exclusive prefix
      double sm = pm, se = pe;
      for (int o = 1; o < 32; o <<= 1) {
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
  };
  if (POST) {
    if (wid < 2) {
      const int r = twist_of(wid);
      if (lane == 0) S.rr[wid] = r;
    }
    __syncthreads();
    scan_from_lanes(wid & 1, wid >> 1, S.rr[wid & 1]);
  } else {
    for (int side = wid; side < NPROBE; side += 3) {
      if (side >= 2 && !has_int) break;
      const int r = twist_of(side);
      scan_from(side, 0, r);
      scan_from(side, 1, r);
    }
  }
  __syncthreads();
  if (tid == 0) atomicMax(&A.ctr[5], (unsigned long long)(clock64() - clk_p1));
  const long long clk_p2 = clock64();

  // ---- phase 3: growth of the candidates, raw and weighted (96 threads;
  // with POST the seventh row -- the interior candidate, ADJ only -- was not
  // written, and its sums are not used for ADJ = 0)
  constexpr int NCG = POST ? 6 : kNC;
  double g[kNC], nl[kNC], nr[kNC], dnl = 0.0, dnr = 0.0;
  double na = 0.0, nbb = 0.0, dna = 0.0, dnb = 0.0;
  unsigned okm = (1u << kNC) - 1u;
  const double *zl = zz[0], *zr = zz[1];
#pragma unroll
  for (int k = 0; k < kNC; ++k) { g[k] = 0.0; nl[k] = 0.0; nr[k] = 0.0; }
#pragma unroll 2
  constexpr int NT = POST ? 128 : 96;  // POST: all four warps (the sums in another order: ulps of a weight)
  for (int i = tid; i < nb; i += NT) {
    const double a = zl[i], b = zr[i];
    const double a2 = a * a, b2 = b * b;
    dnl += a2; dnr += b2;
#pragma unroll
    for (int k = 0; k < NCG; ++k) {
      const double ad = cs_absdplus_fast(TP, QK, zs, k, i);
      if (!(isfinite(ad) && ad != 0.0)) okm &= ~(1u << k);
      g[k] = fmax(g[k], ad);
      nl[k] = fma(ad, a2, nl[k]);
      nr[k] = fma(ad, b2, nr[k]);
      if (ADJ && k == 6 && has_int) {
        const double x = zz[2][i], y = zz[3][i];
        na = fma(ad, x * x, na); nbb = fma(ad, y * y, nbb);
        dna = fma(x, x, dna); dnb = fma(y, y, dnb);
      }
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
    if (ADJ) {
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nbb += __shfl_xor_sync(0xffffffffu, nbb, o);
      dna += __shfl_xor_sync(0xffffffffu, dna, o);
      dnb += __shfl_xor_sync(0xffffffffu, dnb, o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kNC; ++k) {
      S.red[wid][k] = g[k]; S.red[wid][kNC + k] = nl[k]; S.red[wid][2 * kNC + k] = nr[k];
    }
    S.red[wid][3 * kNC] = dnl; S.red[wid][3 * kNC + 1] = dnr;
    S.red[wid][3 * kNC + 2] = na; S.red[wid][3 * kNC + 3] = nbb;
    S.am2[wid][0] = dna; S.am2[wid][1] = dnb;
    S.okw[wid] = okm;
  }
  __syncthreads();

  // ---- phase 4: the tiered choice (readings 9, 30) by thread 0
  if (tid == 0) {
    atomicMax(&A.ctr[6], (unsigned long long)(clock64() - clk_p2));
    double G[kNC], NL[kNC], NR[kNC], DNL = 0.0, DNR = 0.0, NA = 0.0, NB = 0.0, DNA = 0.0, DNB = 0.0;
    unsigned ok = (1u << kNC) - 1u;
    for (int k = 0; k < kNC; ++k) { G[k] = 0.0; NL[k] = 0.0; NR[k] = 0.0; }
    for (int w = 0; w < NT / 32; ++w) {
      for (int k = 0; k < kNC; ++k) {
        G[k] = fmax(G[k], S.red[w][k]);
        NL[k] += S.red[w][kNC + k];
        NR[k] += S.red[w][2 * kNC + k];
      }
      DNL += S.red[w][3 * kNC]; DNR += S.red[w][3 * kNC + 1];
      NA += S.red[w][3 * kNC + 2]; NB += S.red[w][3 * kNC + 3];
      DNA += S.am2[w][0]; DNB += S.am2[w][1];
      ok &= S.okw[w];
    }
    const double spd = P.spdiam;
    int b1 = -1, b2 = -1, b3 = -1;
    int b_int = -1;
    if (has_int && ((ok >> 6) & 1u)) {
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
  for (int i = tid; i < nb; i += (POST ? 128 : 96)) {
    const double Dp = cs_dplus(TP, QK, zs, best, i);
    const double lld = (i < nb - 1) ? __ldg(&LD[i]).y / Dp : 0.0;
    bad |= !isfinite(Dp) || Dp == 0.0 || !isfinite(lld);
    out[i] = make_double2(Dp, lld);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) A.fail[0] = 1;
}

}  // namespace mrrr
