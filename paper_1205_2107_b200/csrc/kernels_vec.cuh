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
// This header holds the per-row arithmetic; the kernels that drive it in
// warp lockstep are in kernels_warp.cuh.
#pragma once
#include "common.cuh"

namespace mrrr {

constexpr int kSeg = MRRR_SEG;

struct VecTask {
  int32_t slot;   // slot id (for lo/hi/j)
  int32_t node;
  int64_t col;    // output column (Z) or scratch vector index
  double lam0;    // starting shift; NaN -> midpoint of [lo, hi]
};

struct FwdCk { double p, q, H; int neg; int pad; };
struct BwdCk { double a, b, K; int neg; int pad; };

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
  // as step(), rescale decided at compile time by the caller (row i with i & 7 == 7)
  __device__ __forceinline__ void step_r(const Row &R, double lam, bool rescale) {
    double t = fma(R.D, q, p);
    neg += negbit(t, q);
    H = R.LD2 * fma(q, q, H);
    p = fma(-lam, t, R.LLD * p);
    q = t;
    if (rescale) fwd_rescale(p, q, H);
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
  __device__ __forceinline__ void step_r(const Row &R, double lam, bool rescale) {
    double u = fma(R.LLD, b, a);
    neg += negbit(u, b);
    K = R.LD2 * fma(b, b, K);
    a = fma(-lam, u, R.D * a);
    b = u;
    if (rescale) bwd_rescale(a, b, K);
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

}  // namespace mrrr
