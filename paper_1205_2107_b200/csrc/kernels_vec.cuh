// kernels_vec.cuh -- a6: singleton eigenvectors by Rayleigh-quotient
// correction on twisted factorizations (
// SURVEY §8(c) O10), one thread per eigenpair.
//
// Projective (division-free) twisted factorization of L D L^T - lambda I
// (DESIGN.md §4.3).  Rows i = 0..nb-1 of the node:
//   stationary (top-down), state before row i: S_i = p_i / q_i,
//     t_i = D_i q_i + p_i (= D+_i q_i), p_{i+1} = LLD_i p_i - lambda t_i, q_{i+1} = t_i,
//     H_{i+1} = LD_i^2 (H_i + q_i^2)        [H_r / q_r^2 = sum_{k<r} z_k^2, z_r = 1]
//   progressive (bottom-up), state at row i: P_i = a_i / b_i,
//     u_{i+1} = LLD_i b_{i+1} + a_{i+1} (= D-_{i+1} b_{i+1}),
//     a_i = D_i a_{i+1} - lambda u_{i+1}, b_i = u_{i+1},
//     K_i = LD_i^2 (K_{i+1} + b_{i+1}^2)     [K_r / b_r^2 = sum_{k>r} z_k^2]
//   twist: gamma_i = S_i + P_i + lambda = N_i / (q_i b_i),
//     N_i = p_i b_i + a_i q_i + lambda q_i b_i;  r = argmin |gamma_i| compared by
//     cross-multiplication (scale-free, no division).
//   solve: z_r = 1, z_i = -LD_i (q_i / t_i) z_{i+1} (i < r),
//          z_{i+1} = -LD_i (b_{i+1} / u_{i+1}) z_i (i >= r).
// Only segment checkpoints (every MRRR_SEG rows) go to global memory; each
// segment is replayed into shared memory when the opposite sweep needs it.
#pragma once
#include "common.cuh"

namespace mrrr {

constexpr int kSeg = MRRR_SEG;
constexpr int kVecThreads = 64;

struct VecTask {
  int32_t slot;   // slot id (for lo/hi/j)
  int32_t node;
  int64_t col;    // output column (Z) or scratch vector index
  double lam0;    // starting shift; NaN -> midpoint of [lo, hi]
};

struct FwdCk { double p, q, H; int neg; int pad; };
struct BwdCk { double a, b; };

struct VecCtx {
  const double2 *DL;   // node (D, LLD)
  const double2 *LDv;  // block (LD, LD^2), offset to the block's first row
  int nb;
  int nseg;
  FwdCk *fck;          // [nseg] stride ntask
  BwdCk *bck;
  int64_t ck_stride;
};

__device__ __forceinline__ void fwd_rescale(double &p, double &q, double &H) {
  int e = max_exp(p, q);
  double f = pow2_scale(min(e, 2045));
  p *= f; q *= f; H = fmin(H * f * f, 1e300);
}
__device__ __forceinline__ void bwd_rescale(double &a, double &b, double &K) {
  int e = max_exp(a, b);
  double f = pow2_scale(min(e, 2045));
  a *= f; b *= f; K = fmin(K * f * f, 1e300);
}

// Result of one twisted factorization
struct Twist {
  int r;
  double gamma;
  double nrm2;
  int negc;
  bool ok;
};

// Full factorization: forward sweep with checkpoints, then backward sweep with
// segment replay and argmin over all twists.  Stores backward checkpoints too.
__device__ Twist twist_full(const VecCtx &X, double lam, int64_t tix, double *smA, double *smB,
                            double *smC) {
  const int T = blockDim.x, tid = threadIdx.x;
  // ---- forward sweep (stationary), checkpoints at segment starts
  double p = -lam, q = 1.0, H = 0.0;
  int neg = 0;
  bool ok = true;
  for (int c = 0; c < X.nseg; ++c) {
    FwdCk ck; ck.p = p; ck.q = q; ck.H = H; ck.neg = neg; ck.pad = 0;
    X.fck[(int64_t)c * X.ck_stride + tix] = ck;
    int r0 = c * kSeg, r1 = min(r0 + kSeg, X.nb - 1);
    for (int i = r0; i < r1; ++i) {
      double2 v = __ldg(&X.DL[i]);
      double ld2 = __ldg(&X.LDv[i]).y;
      double t = fma(v.x, q, p);
      neg += negbit(t, q);
      H = ld2 * fma(q, q, H);
      p = fma(-lam, t, v.y * p);
      q = t;
      if ((i & 7) == 7) fwd_rescale(p, q, H);
    }
  }
  ok &= isfinite(p) && isfinite(q);
  // ---- backward sweep (progressive) with replay of the forward segments
  double a = __ldg(&X.DL[X.nb - 1]).x - lam, b = 1.0, K = 0.0;
  int negB = 0;
  int best_r = X.nb - 1;
  double bN = 0, bden = 0, bH = 0, bq = 1, bK = 0, bb = 1;
  int bneg = 0;
  bool have = false;
  for (int c = X.nseg - 1; c >= 0; --c) {
    int r0 = c * kSeg, r1 = min(r0 + kSeg, X.nb);  // rows [r0, r1)
    // backward checkpoint: state at row min(r0 + kSeg, nb - 1)
    {
      BwdCk bk; bk.a = a; bk.b = b;
      X.bck[(int64_t)c * X.ck_stride + tix] = bk;
    }
    // replay forward rows r0..r1-1 -> (p_i, q_i, H_i) before row i
    FwdCk ck = X.fck[(int64_t)c * X.ck_stride + tix];
    double fp = ck.p, fq = ck.q, fH = ck.H;
    unsigned mask = 0;
    for (int i = r0; i < r1; ++i) {
      int k = i - r0;
      smA[k * T + tid] = fp; smB[k * T + tid] = fq; smC[k * T + tid] = fH;
      if (i < X.nb - 1) {
        double2 v = __ldg(&X.DL[i]);
        double ld2 = __ldg(&X.LDv[i]).y;
        double t = fma(v.x, fq, fp);
        mask |= negbit(t, fq) << k;
        fH = ld2 * fma(fq, fq, fH);
        fp = fma(-lam, t, v.y * fp);
        fq = t;
        if ((i & 7) == 7) fwd_rescale(fp, fq, fH);
      }
    }
    // the top row of the segment: if r1-1 < nb-1 the backward state is at
    // row r1 (= checkpoint row); step down to r1-1 first.
    int top = r1 - 1;
    if (top < X.nb - 1) {
      // state currently at row top+1; step to row top
      double2 v = __ldg(&X.DL[top]);
      double ld2 = __ldg(&X.LDv[top]).y;
      double u = fma(v.y, b, a);
      negB += negbit(u, b);
      K = ld2 * fma(b, b, K);
      a = fma(-lam, u, v.x * a);
      b = u;
      if ((top & 7) == 0) bwd_rescale(a, b, K);
    }
    for (int i = top; i >= r0; --i) {
      int k = i - r0;
      double fpi = smA[k * T + tid], fqi = smB[k * T + tid];
      double qb = fqi * b;
      double N = fma(fpi, b, fma(a, fqi, lam * qb));
      // |N / qb| <= |bN / bden|  <=>  |N| |bden| <= |bN| |qb|  (ties -> smaller i)
      bool better = !have || (fabs(N) * fabs(bden) <= fabs(bN) * fabs(qb));
      if (better && qb != 0.0 && isfinite(N)) {
        have = true;
        best_r = i; bN = N; bden = qb; bH = smC[k * T + tid]; bq = fqi; bK = K; bb = b;
        int negF = ck.neg + __popc(mask & ((1u << k) - 1u));
        bneg = negF + negB;
      }
      if (i > r0) {
        double2 v = __ldg(&X.DL[i - 1]);
        double ld2 = __ldg(&X.LDv[i - 1]).y;
        double u = fma(v.y, b, a);
        negB += negbit(u, b);
        K = ld2 * fma(b, b, K);
        a = fma(-lam, u, v.x * a);
        b = u;
        if (((i - 1) & 7) == 0) bwd_rescale(a, b, K);
      }
    }
  }
  ok &= isfinite(a) && isfinite(b) && have;
  Twist tw;
  tw.r = best_r;
  tw.gamma = bN / bden;
  tw.nrm2 = 1.0 + bH / (bq * bq) + bK / (bb * bb);
  tw.negc = bneg + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = ok && isfinite(tw.gamma) && isfinite(tw.nrm2);
  return tw;
}

// Fixed-twist factorization: forward rows 0..r-1 and backward rows nb-1..r,
// interleaved, with checkpoints for the z pass.
__device__ Twist twist_fixed(const VecCtx &X, double lam, int r, int64_t tix) {
  double p = -lam, q = 1.0, H = 0.0;
  int negF = 0;
  double a = __ldg(&X.DL[X.nb - 1]).x - lam, b = 1.0, K = 0.0;
  int negB = 0;
  int nf = r;               // forward steps: rows 0..r-1
  int nbk = X.nb - 1 - r;   // backward steps: rows nb-2 down to r
  int steps = max(nf, nbk);
  int cseg_top = X.nseg - 1;
  // the first backward checkpoint (top segment) is the initial state
  for (int s = 0; s < steps; ++s) {
    if (s < nf) {
      int i = s;
      if ((i % kSeg) == 0) {
        FwdCk ck; ck.p = p; ck.q = q; ck.H = H; ck.neg = negF; ck.pad = 0;
        X.fck[(int64_t)(i / kSeg) * X.ck_stride + tix] = ck;
      }
      double2 v = __ldg(&X.DL[i]);
      double ld2 = __ldg(&X.LDv[i]).y;
      double t = fma(v.x, q, p);
      negF += negbit(t, q);
      H = ld2 * fma(q, q, H);
      p = fma(-lam, t, v.y * p);
      q = t;
      if ((i & 7) == 7) fwd_rescale(p, q, H);
    }
    if (s < nbk) {
      int i = X.nb - 2 - s;  // step from row i+1 to row i
      // backward checkpoint c holds the state at row min((c+1) kSeg, nb-1)
      int ra = i + 1;
      BwdCk bk; bk.a = a; bk.b = b;
      if (ra == X.nb - 1) {
        X.bck[(int64_t)cseg_top * X.ck_stride + tix] = bk;
        if ((ra % kSeg) == 0 && cseg_top >= 1)
          X.bck[(int64_t)(cseg_top - 1) * X.ck_stride + tix] = bk;
      } else if ((ra % kSeg) == 0) {
        X.bck[(int64_t)(ra / kSeg - 1) * X.ck_stride + tix] = bk;
      }
      double2 v = __ldg(&X.DL[i]);
      double ld2 = __ldg(&X.LDv[i]).y;
      double u = fma(v.y, b, a);
      negB += negbit(u, b);
      K = ld2 * fma(b, b, K);
      a = fma(-lam, u, v.x * a);
      b = u;
      if ((i & 7) == 0) bwd_rescale(a, b, K);
    }
  }
  double qb = q * b;
  double N = fma(p, b, fma(a, q, lam * qb));
  Twist tw;
  tw.r = r;
  tw.gamma = N / qb;
  tw.nrm2 = 1.0 + H / (q * q) + K / (b * b);
  tw.negc = negF + negB + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = isfinite(tw.gamma) && isfinite(tw.nrm2) && qb != 0.0;
  return tw;
}

// z pass: z_r = 1; write scale * z_i to out[i * ostride] for all rows.
__device__ void twist_solve(const VecCtx &X, double lam, int r, double scale, double *out,
                            int64_t ostride, int64_t tix, double *smA, double *smB) {
  const int T = blockDim.x, tid = threadIdx.x;
  out[(int64_t)r * ostride] = scale;
  // left part, i < r, descending: z_i = -LD_i (q_i / t_i) z_{i+1}
  double z1 = 1.0, z2 = 0.0;  // z_{i+1}, z_{i+2}
  if (r > 0) {
    int clast = (r - 1) / kSeg;
    for (int c = clast; c >= 0; --c) {
      int r0 = c * kSeg, r1 = min(r0 + kSeg, r);  // rows [r0, r1) all < r
      FwdCk ck = X.fck[(int64_t)c * X.ck_stride + tix];
      double fp = ck.p, fq = ck.q, fH = ck.H;
      for (int i = r0; i < r1; ++i) {
        double2 v = __ldg(&X.DL[i]);
        double t = fma(v.x, fq, fp);
        smA[(i - r0) * T + tid] = fq;
        smB[(i - r0) * T + tid] = t;
        fp = fma(-lam, t, v.y * fp);
        fq = t;
        if ((i & 7) == 7) { double dummy = 0; fwd_rescale(fp, fq, dummy); }
      }
      (void)fH;
      for (int i = r1 - 1; i >= r0; --i) {
        double ld = __ldg(&X.LDv[i]).x;
        double zi;
        if (z1 != 0.0) {
          zi = -ld * z1 * (smA[(i - r0) * T + tid] / smB[(i - r0) * T + tid]);
        } else {
          zi = -(__ldg(&X.LDv[i + 1]).x / ld) * z2;
        }
        if (!(fabs(zi) >= kTiny)) zi = 0.0;
        out[(int64_t)i * ostride] = zi * scale;
        z2 = z1; z1 = zi;
      }
    }
  }
  // right part, i > r, ascending: z_{i+1} = -LD_i (b_{i+1} / u_{i+1}) z_i
  double y1 = 1.0, y2 = 0.0;  // z_i, z_{i-1}
  if (r < X.nb - 1) {
    int cfirst = r / kSeg;
    for (int c = cfirst; c < X.nseg; ++c) {
      int r0 = c * kSeg;
      int top = min(r0 + kSeg, X.nb - 1);  // checkpoint row
      int lo_i = max(r0, r);                // rows i in [lo_i, top) give U-_i
      if (lo_i >= top) continue;
      BwdCk bk = X.bck[(int64_t)c * X.ck_stride + tix];
      double a = bk.a, b = bk.b, K = 0.0;
      for (int i = top - 1; i >= lo_i; --i) {
        double2 v = __ldg(&X.DL[i]);
        double u = fma(v.y, b, a);
        smA[(i - r0) * T + tid] = b;  // b_{i+1}
        smB[(i - r0) * T + tid] = u;  // u_{i+1}
        a = fma(-lam, u, v.x * a);
        b = u;
        if ((i & 7) == 0) bwd_rescale(a, b, K);
      }
      for (int i = lo_i; i < top; ++i) {
        double ld = __ldg(&X.LDv[i]).x;
        double zn;
        if (y1 != 0.0) {
          zn = -ld * y1 * (smA[(i - r0) * T + tid] / smB[(i - r0) * T + tid]);
        } else {
          zn = -(__ldg(&X.LDv[i - 1]).x / ld) * y2;
        }
        if (!(fabs(zn) >= kTiny)) zn = 0.0;
        out[(int64_t)(i + 1) * ostride] = zn * scale;
        y2 = y1; y1 = zn;
      }
    }
  }
}

struct VecArgs {
  const Node *nodes;
  const Block *blocks;
  const double2 *LDv;        // global (LD, LD^2) per row
  const VecTask *tasks;
  int ntask;
  const double *lo, *hi;     // slot brackets (node coordinates)
  const int *slot_j;
  FwdCk *fck;
  BwdCk *bck;
  int64_t ck_stride;
  int nseg_max;
  // outputs
  double *Z; int64_t ldz;    // mode 0
  double *lam_out;           // mode 0: final lambda in node coordinates per task
  double *zbuf; int64_t zstride;  // mode 1
  int mode;                  // 0 = RQC + normalised Z column, 1 = one pass to zbuf
  double rtol_fallback;
  unsigned long long *ctr;   // [0] factorizations, [1] fallbacks, [2] nudges
  int *task_info;            // optional: per task (iterations | fallback << 8)
  int trace_task;            // task id whose RQC trajectory is printed (-1: none)
};

__device__ __forceinline__ void vectors_body(const VecArgs &A) {
  extern __shared__ double smv[];
  const int T = blockDim.x;
  double *smA = smv, *smB = smv + kSeg * T, *smC = smv + 2 * kSeg * T;
  int tix = blockIdx.x * blockDim.x + threadIdx.x;
  if (tix >= A.ntask) return;
  VecTask tk = A.tasks[tix];
  const Node N = A.nodes[tk.node];
  VecCtx X;
  X.DL = N.DL;
  X.LDv = A.LDv + N.row0;
  X.nb = N.nb;
  X.nseg = (N.nb + kSeg - 1) / kSeg;
  X.fck = A.fck; X.bck = A.bck; X.ck_stride = A.ck_stride;
  double lo = A.lo[tk.slot], hi = A.hi[tk.slot];
  int j = A.slot_j[tk.slot];
  unsigned long long nfact = 0, nudges = 0, fb = 0;

  if (N.nb == 1) {
    double lamf = __ldg(&N.DL[0]).x;
    if (A.mode == 0) {
      A.Z[tk.col * A.ldz + N.row0] = 1.0;
      A.lam_out[tix] = lamf;
    } else {
      A.zbuf[tk.col * A.zstride] = 1.0;
    }
    return;
  }

  double lam = isnan(tk.lam0) ? 0.5 * (lo + hi) : tk.lam0;
  Twist tw;
  // full factorization; nudge lambda if it is not finite (zero pivots are
  // handled projectively, this is only overflow insurance; reading 25)
  double nudge = 2.0 * kEps * fabs(lam) + kTiny;
  double lam_base = lam;
  for (int tries = 0; tries < 60; ++tries) {
    tw = twist_full(X, lam, tix, smA, smB, smC);
    ++nfact;
    if (tw.ok) break;
    ++nudges;
    lam = lam_base + nudge;
    nudge *= 2.0;
  }
  double lam_fin = lam;
  if (A.mode == 1) {
    double sc = 1.0 / sqrt(tw.nrm2);
    twist_solve(X, lam, tw.r, sc, A.zbuf + tk.col * A.zstride, 1, tix, smA, smB);
    atomicAdd(&A.ctr[0], nfact);
    return;
  }
  bool converged = false;
  int it = 1;
  const bool trace = tix == A.trace_task;
  for (;;) {
    if (tw.negc >= j) { if (lam < hi) hi = lam; } else { if (lam > lo) lo = lam; }
    double delta = tw.gamma / tw.nrm2;
    if (trace)
      printf("[task %d it %d] j %d lam %.17g r %d gamma %.6e nrm2 %.6e delta %.6e negc %d lo %.17g hi %.17g ok %d\n",
             tix, it, j, lam, tw.r, tw.gamma, tw.nrm2, delta, tw.negc, lo, hi, (int)tw.ok);
    if (fabs(delta) <= 4.0 * kEps * fabs(lam) || lam + delta == lam) {
      lam_fin = lam + delta; converged = true; break;
    }
    double nw = lam + delta;
    if (nw <= lo || nw >= hi) {
      if (lam == lo || lam == hi) {
        nw = 0.5 * (lo + hi);
        if (nw <= lo || nw >= hi) { lam_fin = lam; converged = true; break; }
      } else {
        nw = (nw <= lo) ? lo : hi;
      }
    }
    lam = nw;
    if (it >= 10) break;
    Twist t2 = twist_fixed(X, lam, tw.r, tix);
    ++nfact; ++it;
    if (!t2.ok) {
      // fall back to a full factorization at this shift
      t2 = twist_full(X, lam, tix, smA, smB, smC);
      ++nfact;
      if (!t2.ok) break;
    }
    tw = t2;
  }
  if (!converged) {
    // O10 fallback: bisection to 4 eps relative, one final factorization
    ++fb;
    for (int k = 0; k < 200; ++k) {
      double m = 0.5 * (lo + hi);
      if (hi - lo <= A.rtol_fallback * fmax(fabs(lo), fabs(hi)) || !(m > lo && m < hi)) break;
      if ((int)negcount_global(N.DL, N.nb, m, nullptr) >= j) hi = m; else lo = m;
    }
    lam = 0.5 * (lo + hi);
    tw = twist_full(X, lam, tix, smA, smB, smC);
    ++nfact;
    lam_fin = lam;
  }
  double sc = 1.0 / sqrt(tw.nrm2);
  twist_solve(X, lam, tw.r, sc, A.Z + tk.col * A.ldz + N.row0, 1, tix, smA, smB);
  A.lam_out[tix] = lam_fin;
  if (A.task_info) A.task_info[tix] = it | ((int)fb << 8);
  atomicAdd(&A.ctr[0], nfact);
  if (fb) atomicAdd(&A.ctr[1], fb);
  if (nudges) atomicAdd(&A.ctr[2], nudges);
}

// Final singleton vectors (mode 0) and the parent-vector probe of the child
// acceptance test (mode 1) are separate entry points so profiles tell them apart.
__global__ void __launch_bounds__(kVecThreads) k_vectors(VecArgs A) { vectors_body(A); }
__global__ void __launch_bounds__(kVecThreads) k_zprobe(VecArgs A) { vectors_body(A); }

}  // namespace mrrr
