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
//
// Latency: every sweep streams its rows through registers one group of
// kGrp rows ahead of the recurrence (stream_up / stream_down), so the
// dependent fp64 chain does not wait on global loads (ncu on the first
// version: 5.8 long-scoreboard stalls per issue, FP64 pipe 3 % active).
#pragma once
#include "common.cuh"

namespace mrrr {

constexpr int kSeg = MRRR_SEG;
constexpr int kVecThreads = 32;
constexpr int kGrp = 4;  // prefetch group (rows)

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

// One row of the representation as the sweeps need it.
struct Row { double D, LLD, LD, LD2; };

__device__ __forceinline__ Row ldrow(const VecCtx &X, int i) {
  double2 a = __ldg(&X.DL[i]);
  double2 b = __ldg(&X.LDv[i]);
  Row r; r.D = a.x; r.LLD = a.y; r.LD = b.x; r.LD2 = b.y;
  return r;
}

// Calls f(i, row) for i = a, a+1, ..., b-1 (ascending), rows loaded one group
// ahead.
template <class F>
__device__ __forceinline__ void stream_up(const VecCtx &X, int a, int b, F &&f) {
  if (a >= b) return;
  Row cur[kGrp], nxt[kGrp];
#pragma unroll
  for (int k = 0; k < kGrp; ++k) if (a + k < b) cur[k] = ldrow(X, a + k);
  for (int i = a; i < b; i += kGrp) {
#pragma unroll
    for (int k = 0; k < kGrp; ++k) if (i + kGrp + k < b) nxt[k] = ldrow(X, i + kGrp + k);
#pragma unroll
    for (int k = 0; k < kGrp; ++k) if (i + k < b) f(i + k, cur[k]);
#pragma unroll
    for (int k = 0; k < kGrp; ++k) cur[k] = nxt[k];
  }
}

// Calls f(i, row) for i = b, b-1, ..., a (descending, inclusive bounds).
template <class F>
__device__ __forceinline__ void stream_down(const VecCtx &X, int b, int a, F &&f) {
  if (b < a) return;
  Row cur[kGrp], nxt[kGrp];
#pragma unroll
  for (int k = 0; k < kGrp; ++k) if (b - k >= a) cur[k] = ldrow(X, b - k);
  for (int i = b; i >= a; i -= kGrp) {
#pragma unroll
    for (int k = 0; k < kGrp; ++k) if (i - kGrp - k >= a) nxt[k] = ldrow(X, i - kGrp - k);
#pragma unroll
    for (int k = 0; k < kGrp; ++k) if (i - k >= a) f(i - k, cur[k]);
#pragma unroll
    for (int k = 0; k < kGrp; ++k) cur[k] = nxt[k];
  }
}

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

// Stationary step over row i (state before row i -> before row i+1).
struct Fwd {
  double p, q, H;
  int neg;
  __device__ __forceinline__ void step(int i, const Row &R, double lam) {
    double t = fma(R.D, q, p);
    neg += negbit(t, q);
    H = R.LD2 * fma(q, q, H);
    p = fma(-lam, t, R.LLD * p);
    q = t;
    if ((i & 7) == 7) fwd_rescale(p, q, H);
  }
};
// Progressive step into row i from row i+1 (uses row i).
struct Bwd {
  double a, b, K;
  int neg;
  __device__ __forceinline__ void step(int i, const Row &R, double lam) {
    double u = fma(R.LLD, b, a);
    neg += negbit(u, b);
    K = R.LD2 * fma(b, b, K);
    a = fma(-lam, u, R.D * a);
    b = u;
    if ((i & 7) == 0) bwd_rescale(a, b, K);
  }
};

// Result of one twisted factorization
struct Twist {
  int r;
  double gamma;
  double nrm2;
  int negc;
  bool ok;
};

__device__ __forceinline__ void put_fck(const VecCtx &X, int c, int64_t tix, const Fwd &F) {
  FwdCk ck; ck.p = F.p; ck.q = F.q; ck.H = F.H; ck.neg = F.neg; ck.pad = 0;
  X.fck[(int64_t)c * X.ck_stride + tix] = ck;
}

// Full factorization: forward sweep with checkpoints, then backward sweep with
// segment replay and argmin over all twists.  Stores backward checkpoints too.
__device__ __noinline__ Twist twist_full(const VecCtx &X, double lam, int64_t tix, double *smA, double *smB,
                            double *smC) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int nb = X.nb;
  // ---- forward sweep (stationary), checkpoints at segment starts
  Fwd F{-lam, 1.0, 0.0, 0};
  stream_up(X, 0, nb - 1, [&](int i, const Row &R) {
    if (i % kSeg == 0) put_fck(X, i / kSeg, tix, F);
    F.step(i, R, lam);
  });
  if ((nb - 1) % kSeg == 0) put_fck(X, (nb - 1) / kSeg, tix, F);
  bool ok = isfinite(F.p) && isfinite(F.q);
  // ---- backward sweep (progressive) with replay of the forward segments
  Bwd B{__ldg(&X.DL[nb - 1]).x - lam, 1.0, 0.0, 0};
  int best_r = nb - 1;
  double bN = 0, bden = 0, bH = 0, bq = 1, bK = 0, bb = 1;
  int bneg = 0;
  bool have = false;
  for (int c = X.nseg - 1; c >= 0; --c) {
    const int r0 = c * kSeg, r1 = min(r0 + kSeg, nb);  // rows [r0, r1)
    {
      BwdCk bk; bk.a = B.a; bk.b = B.b;  // state at row min(r0 + kSeg, nb - 1)
      X.bck[(int64_t)c * X.ck_stride + tix] = bk;
    }
    // replay forward rows r0..r1-1 -> (p_i, q_i, H_i) before row i and the
    // negative-pivot mask of the segment
    const FwdCk ck = X.fck[(int64_t)c * X.ck_stride + tix];
    Fwd G{ck.p, ck.q, ck.H, 0};
    unsigned mask = 0;
    stream_up(X, r0, min(r1, nb - 1), [&](int i, const Row &R) {
      const int k = i - r0;
      smA[k * T + tid] = G.p; smB[k * T + tid] = G.q; smC[k * T + tid] = G.H;
      const int before = G.neg;
      G.step(i, R, lam);
      mask |= (unsigned)(G.neg - before) << k;
    });
    if (r1 == nb) {  // row nb-1: the state before it
      const int k = nb - 1 - r0;
      smA[k * T + tid] = G.p; smB[k * T + tid] = G.q; smC[k * T + tid] = G.H;
    }
    const int top = r1 - 1;
    auto eval = [&](int i) {
      const int k = i - r0;
      const double fpi = smA[k * T + tid], fqi = smB[k * T + tid];
      const double qb = fqi * B.b;
      const double N = fma(fpi, B.b, fma(B.a, fqi, lam * qb));
      // |N / qb| <= |bN / bden|  <=>  |N| |bden| <= |bN| |qb|  (ties -> smaller i)
      const bool better = !have || (fabs(N) * fabs(bden) <= fabs(bN) * fabs(qb));
      if (better && qb != 0.0 && isfinite(N)) {
        have = true;
        best_r = i; bN = N; bden = qb; bH = smC[k * T + tid]; bq = fqi; bK = B.K; bb = B.b;
        bneg = ck.neg + __popc(mask & ((1u << k) - 1u)) + B.neg;
      }
    };
    int start = top;
    if (top == nb - 1) { eval(top); start = top - 1; }
    stream_down(X, start, r0, [&](int i, const Row &R) {
      B.step(i, R, lam);
      eval(i);
    });
  }
  ok &= isfinite(B.a) && isfinite(B.b) && have;
  Twist tw;
  tw.r = best_r;
  tw.gamma = bN / bden;
  tw.nrm2 = 1.0 + bH / (bq * bq) + bK / (bb * bb);
  tw.negc = bneg + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = ok && isfinite(tw.gamma) && isfinite(tw.nrm2);
  return tw;
}

// Fixed-twist factorization: forward rows 0..r-1 and backward rows nb-2..r as
// two interleaved dependency chains, with checkpoints for the z pass.
__device__ __noinline__ Twist twist_fixed(const VecCtx &X, double lam, int r, int64_t tix) {
  const int nb = X.nb;
  Fwd F{-lam, 1.0, 0.0, 0};
  Bwd B{__ldg(&X.DL[nb - 1]).x - lam, 1.0, 0.0, 0};
  const int nf = r;            // forward steps: rows 0..r-1
  const int nbk = nb - 1 - r;  // backward steps: rows nb-2 down to r
  const int steps = max(nf, nbk);
  const int cseg_top = X.nseg - 1;
  constexpr int G = 4;
  Row fc[G], fn[G], bc[G], bn[G];
#pragma unroll
  for (int k = 0; k < G; ++k) {
    if (k < nf) fc[k] = ldrow(X, k);
    if (k < nbk) bc[k] = ldrow(X, nb - 2 - k);
  }
  for (int s0 = 0; s0 < steps; s0 += G) {
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (s0 + G + k < nf) fn[k] = ldrow(X, s0 + G + k);
      if (s0 + G + k < nbk) bn[k] = ldrow(X, nb - 2 - (s0 + G + k));
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int s = s0 + k;
      if (s < nf) {
        if ((s % kSeg) == 0) put_fck(X, s / kSeg, tix, F);
        F.step(s, fc[k], lam);
      }
      if (s < nbk) {
        const int i = nb - 2 - s;  // step from row i+1 to row i
        // backward checkpoint c holds the state at row min((c+1) kSeg, nb-1)
        const int ra = i + 1;
        BwdCk bk; bk.a = B.a; bk.b = B.b;
        if (ra == nb - 1) {
          X.bck[(int64_t)cseg_top * X.ck_stride + tix] = bk;
          if ((ra % kSeg) == 0 && cseg_top >= 1) X.bck[(int64_t)(cseg_top - 1) * X.ck_stride + tix] = bk;
        } else if ((ra % kSeg) == 0) {
          X.bck[(int64_t)(ra / kSeg - 1) * X.ck_stride + tix] = bk;
        }
        B.step(i, bc[k], lam);
      }
    }
#pragma unroll
    for (int k = 0; k < G; ++k) { fc[k] = fn[k]; bc[k] = bn[k]; }
  }
  const double qb = F.q * B.b;
  const double N = fma(F.p, B.b, fma(B.a, F.q, lam * qb));
  Twist tw;
  tw.r = r;
  tw.gamma = N / qb;
  tw.nrm2 = 1.0 + F.H / (F.q * F.q) + B.K / (B.b * B.b);
  tw.negc = F.neg + B.neg + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = isfinite(tw.gamma) && isfinite(tw.nrm2) && qb != 0.0;
  return tw;
}

// z pass: z_r = 1; write scale * z_i to out[i * ostride] for all rows.
__device__ __noinline__ void twist_solve(const VecCtx &X, double lam, int r, double scale, double *out,
                            int64_t ostride, int64_t tix, double *smA, double *smB, double *smC) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int nb = X.nb;
  out[(int64_t)r * ostride] = scale;
  // left part, i < r, descending: z_i = -LD_i (q_i / t_i) z_{i+1}
  double z1 = 1.0, z2 = 0.0, ldn = 0.0;  // z_{i+1}, z_{i+2}, LD_{i+1}
  if (r > 0) {
    ldn = __ldg(&X.LDv[r]).x;
    const int clast = (r - 1) / kSeg;
    for (int c = clast; c >= 0; --c) {
      const int r0 = c * kSeg, r1 = min(r0 + kSeg, r);  // rows [r0, r1) all < r
      const FwdCk ck = X.fck[(int64_t)c * X.ck_stride + tix];
      Fwd G{ck.p, ck.q, 0.0, 0};
      stream_up(X, r0, r1, [&](int i, const Row &R) {
        const int k = i - r0;
        const double t = fma(R.D, G.q, G.p);
        smA[k * T + tid] = G.q;
        smB[k * T + tid] = t;
        smC[k * T + tid] = R.LD;
        G.p = fma(-lam, t, R.LLD * G.p);
        G.q = t;
        if ((i & 7) == 7) fwd_rescale(G.p, G.q, G.H);
      });
      for (int i = r1 - 1; i >= r0; --i) {
        const int k = i - r0;
        const double ld = smC[k * T + tid];
        double zi;
        if (z1 != 0.0) {
          zi = -ld * z1 * (smA[k * T + tid] / smB[k * T + tid]);
        } else {
          zi = -(ldn / ld) * z2;  // row i+1 of (LDL^T - lambda I) z = 0
        }
        if (!(fabs(zi) >= kTiny)) zi = 0.0;
        out[(int64_t)i * ostride] = zi * scale;
        z2 = z1; z1 = zi; ldn = ld;
      }
    }
  }
  // right part, i > r, ascending: z_{i+1} = -LD_i (b_{i+1} / u_{i+1}) z_i
  double y1 = 1.0, y2 = 0.0;  // z_i, z_{i-1}
  double ldp = (r > 0) ? __ldg(&X.LDv[r - 1]).x : 0.0;  // LD_{i-1}
  if (r < nb - 1) {
    const int cfirst = r / kSeg;
    for (int c = cfirst; c < X.nseg; ++c) {
      const int r0 = c * kSeg;
      const int top = min(r0 + kSeg, nb - 1);  // checkpoint row
      const int lo_i = max(r0, r);              // rows i in [lo_i, top) give U-_i
      if (lo_i >= top) continue;
      const BwdCk bk = X.bck[(int64_t)c * X.ck_stride + tix];
      Bwd G{bk.a, bk.b, 0.0, 0};
      stream_down(X, top - 1, lo_i, [&](int i, const Row &R) {
        const int k = i - r0;
        const double u = fma(R.LLD, G.b, G.a);
        smA[k * T + tid] = G.b;  // b_{i+1}
        smB[k * T + tid] = u;    // u_{i+1}
        smC[k * T + tid] = R.LD;
        G.a = fma(-lam, u, R.D * G.a);
        G.b = u;
        if ((i & 7) == 0) bwd_rescale(G.a, G.b, G.K);
      });
      for (int i = lo_i; i < top; ++i) {
        const int k = i - r0;
        const double ld = smC[k * T + tid];
        double zn;
        if (y1 != 0.0) {
          zn = -ld * y1 * (smA[k * T + tid] / smB[k * T + tid]);
        } else {
          zn = -(ldp / ld) * y2;  // row i of (LDL^T - lambda I) z = 0
        }
        if (!(fabs(zn) >= kTiny)) zn = 0.0;
        out[(int64_t)(i + 1) * ostride] = zn * scale;
        y2 = y1; y1 = zn; ldp = ld;
      }
    }
  }
}

struct VecArgs {
  const Node *nodes;
  const Block *blocks;
  const double2 *LDv;        // global (LD, LD^2) per row
  const VecTask *tasks;
  const int *task_list;      // optional indirection (fallback pass); nullptr = identity
  int ntask;                 // tasks (or list entries) to process
  double *lo, *hi;           // slot brackets (node coordinates)
  const int *slot_j;
  FwdCk *fck;
  BwdCk *bck;
  int64_t ck_stride;
  int nseg_max;
  // outputs
  double *Z; int64_t ldz;    // modes 0 and 2
  double *lam_out;           // modes 0 and 2: final lambda in node coordinates per task
  double *zbuf; int64_t zstride;  // mode 1
  int mode;                  // 0 = RQC + normalised Z column; 1 = one pass to zbuf;
                             // 2 = one factorization at the bracket midpoint + Z column
                             //     (after the fallback bisection)
  int *fail_list;            // mode 0: tasks whose RQC did not converge (appended)
  int *fail_count;
  unsigned long long *ctr;   // [0] factorizations, [1] fallbacks, [2] nudges
  int *task_info;            // optional: per task (iterations | fallback << 8)
  int trace_task;            // task id whose RQC trajectory is printed (-1: none)
};

__device__ __forceinline__ void vectors_body(const VecArgs &A) {
  extern __shared__ double smv[];
  const int T = blockDim.x;
  double *smA = smv, *smB = smv + kSeg * T, *smC = smv + 2 * kSeg * T;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= A.ntask) return;
  const int tix = A.task_list ? A.task_list[q] : q;
  const VecTask tk = A.tasks[tix];
  const Node N = A.nodes[tk.node];
  VecCtx X;
  X.DL = N.DL;
  X.LDv = A.LDv + N.row0;
  X.nb = N.nb;
  X.nseg = (N.nb + kSeg - 1) / kSeg;
  X.fck = A.fck; X.bck = A.bck; X.ck_stride = A.ck_stride;
  double lo = A.lo[tk.slot], hi = A.hi[tk.slot];
  const int j = A.slot_j[tk.slot];
  unsigned long long nfact = 0, nudges = 0;

  if (N.nb == 1) {
    const double lamf = __ldg(&N.DL[0]).x;
    if (A.mode != 1) {
      A.Z[tk.col * A.ldz + N.row0] = 1.0;
      A.lam_out[tix] = lamf;
    } else {
      A.zbuf[tk.col * A.zstride] = 1.0;
    }
    return;
  }

  double lam = (A.mode == 2 || isnan(tk.lam0)) ? 0.5 * (lo + hi) : tk.lam0;
  Twist tw;
  // full factorization; nudge lambda if it is not finite (zero pivots are
  // handled projectively, this is only overflow insurance; reading 25)
  double nudge = 2.0 * kEps * fabs(lam) + kTiny;
  const double lam_base = lam;
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
    const double sc = 1.0 / sqrt(tw.nrm2);
    twist_solve(X, lam, tw.r, sc, A.zbuf + tk.col * A.zstride, 1, tix, smA, smB, smC);
    atomicAdd(&A.ctr[0], nfact);
    return;
  }
  int it = 1;
  if (A.mode == 0) {
    bool converged = false;
    const bool trace = tix == A.trace_task;
    for (;;) {
      if (tw.negc >= j) { if (lam < hi) hi = lam; } else { if (lam > lo) lo = lam; }
      const double delta = tw.gamma / tw.nrm2;
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
      // O10 fallback, deferred: the bracket goes back to the slot, a
      // CTA-parallel multisection (k_fallback_bisect) refines it to 4 eps and
      // a mode-2 pass writes the vector.
      A.lo[tk.slot] = lo; A.hi[tk.slot] = hi;
      A.fail_list[atomicAdd(A.fail_count, 1)] = tix;
      atomicAdd(&A.ctr[0], nfact);
      atomicAdd(&A.ctr[1], 1ull);
      if (A.task_info) A.task_info[tix] = it | (1 << 8);
      return;
    }
  }
  const double sc = 1.0 / sqrt(tw.nrm2);
  twist_solve(X, lam, tw.r, sc, A.Z + tk.col * A.ldz + N.row0, 1, tix, smA, smB, smC);
  A.lam_out[tix] = lam_fin;
  atomicAdd(&A.ctr[0], nfact);
  if (nudges) atomicAdd(&A.ctr[2], nudges);
  if (A.task_info && A.mode == 0) A.task_info[tix] = it;
}

// Final singleton vectors (modes 0, 2) and the parent-vector probe of the
// child acceptance test (mode 1) are separate entry points so profiles tell
// them apart.
__global__ void __launch_bounds__(kVecThreads) k_vectors(VecArgs A) { vectors_body(A); }
__global__ void __launch_bounds__(kVecThreads) k_zprobe(VecArgs A) { vectors_body(A); }

}  // namespace mrrr
