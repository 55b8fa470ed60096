// kernels_warp.cuh -- a6: twisted factorizations and eigenvector solves in
// WARP LOCKSTEP.  A work item is up to 32 eigenpairs of ONE node (one lane
// each); all lanes walk the node's rows in the same order, so the rows are
// staged once per warp through a shared-memory ring of 16-row tiles filled
// by cp.async (LDGSTS) kRing-1 tiles ahead, and read back as broadcasts.
// Measured on B200 (tools/ubench_chain.cu): a dependent projective sweep
// costs 37 cycles/row from such tiles against 72-80 from global memory with
// register prefetch, and 26.5 with rows in registers.
//
// Arithmetic is that of kernels_vec.cuh: projective
// stationary/progressive transforms, twist by cross-multiplied |gamma|,
// running partial norms H/K, checkpoints every kTR rows with replay.  Each
// item runs on a PAIR of warps (stationary sweeps on one, progressive on the
// other, concurrently; see below).  The eigenvector z of each lane is formed
// per segment in shared memory and written to its column with 16-byte stores.
#pragma once
#include <cuda_pipeline.h>

#include "kernels_vec.cuh"

namespace mrrr {

constexpr int kTR = 16;          // rows per tile (= checkpoint segment)
#ifndef MRRR_VRING
#define MRRR_VRING 6
#endif
constexpr int kRing = MRRR_VRING;  // tiles in flight per warp
static_assert(kTR == kSeg, "tiles and checkpoint segments coincide");

// A work item may hold the eigenpairs of up to kMaxSeg nodes ("segments") of
// one block: the nodes of a block share the row count, the first row and the
// (LD, LD^2) rows (LD is invariant under the stationary transform), and
// differ only in (D, LLD).  Packing the singletons of several small nodes
// into one warp keeps the lanes busy: deep tree levels deliver a few
// singletons per node, and one node per warp left ~79 % of the lanes idle at
// n = 20000 (3000 items for 20000 eigenpairs).
#ifndef MRRR_VSEG
#define MRRR_VSEG 8
#endif
constexpr int kMaxSeg = MRRR_VSEG;

// Shared memory of one warp.
struct WarpSmem {
  double2 rDL[kRing][kTR][kMaxSeg];  // (D, LLD) rows of each segment's node
  double2 rLD[kRing][kTR];           // (LD, LD^2) rows (shared by the block's nodes)
  double sA[kTR][32], sB[kTR][32], sC[kTR][32];  // per-lane segment stores (z goes to sA)
  const double2 *segDL[kMaxSeg];     // (D, LLD) array of each segment's node
};

constexpr int kCpMax = (kMaxSeg + 2) / 2;  // ring copies per lane per tile (segments h, h+2, .. <= nsegs)

struct WarpCtx {
  const double2 *DL, *LDv;  // DL: this lane's node
  int nb, nseg, lane;
  int seg, nsegs;           // this lane's segment; segments of the item
  const double2 *cp_src[kCpMax];  // this lane's ring copies: sources of segments h + 2j (h = lane / 16)
  int cp_n;
  WarpSmem *sm;
  FwdCk *fck;
  BwdCk *bck;
  int64_t ck_stride, tix;  // checkpoint column of this lane
};

__device__ __forceinline__ void w_issue(const WarpCtx &W, int c, int slot) {
  // copies 16 (D, LLD) rows per segment, then the 16 (LD, LD^2) rows: lane l
  // copies row l % 16 of segments l / 16, l / 16 + 2, ... (the (LD, LD^2)
  // rows count as segment nsegs); the sources were resolved once per item
  // (w_segments), so a tile costs a few predicated copies per lane
  if (c >= 0 && c < W.nseg) {
    const int k = W.lane & (kTR - 1), h = W.lane >> 4;
    const int row = c * kTR + k;
    if (row < W.nb) {
#pragma unroll
      for (int j = 0; j < kCpMax; ++j) {
        const int sg = h + 2 * j;
        if (j < W.cp_n) {
          if (sg < W.nsegs) __pipeline_memcpy_async(&W.sm->rDL[slot][k][sg], W.cp_src[j] + row, sizeof(double2));
          else __pipeline_memcpy_async(&W.sm->rLD[slot][k], W.cp_src[j] + row, sizeof(double2));
        }
      }
    }
  }
  __pipeline_commit();
}

// Segment structure of an item: lanes whose tasks (in position order t0 ..
// t1-1) share a node form a segment; idle lanes join the last one.  The
// first lane of each segment publishes its node's (D, LLD) array.
__device__ __forceinline__ void w_segments(WarpCtx &W, int node_at_pos, bool active) {
  const int prev = __shfl_up_sync(0xffffffffu, node_at_pos, 1);
  const bool first = W.lane == 0 || (active && node_at_pos != prev);
  const unsigned b = __ballot_sync(0xffffffffu, first);
  W.seg = __popc(b & (0xffffffffu >> (31 - W.lane))) - 1;
  W.nsegs = __popc(b);
  if (first) W.sm->segDL[W.seg] = W.DL;
  __syncwarp();
  const int h = W.lane >> 4;
  W.cp_n = W.nsegs >= h ? (W.nsegs - h) / 2 + 1 : 0;
#pragma unroll
  for (int j = 0; j < kCpMax; ++j) {
    const int sg = h + 2 * j;
    W.cp_src[j] = sg < W.nsegs ? W.sm->segDL[sg] : W.LDv;
  }
}

// f(c, slot) for tiles c = c0 .. c1 (ascending, warp-uniform bounds); tile c
// is in ring slot `slot` when f runs.
template <class F>
__device__ __forceinline__ void w_tiles_up(const WarpCtx &W, int c0, int c1, F &&f) {
  if (c0 > c1) return;
#pragma unroll
  for (int k = 0; k < kRing - 1; ++k) w_issue(W, c0 + k <= c1 ? c0 + k : -1, (c0 + k) % kRing);
  for (int c = c0; c <= c1; ++c) {
    __pipeline_wait_prior(kRing - 2);
    __syncwarp();
    f(c, c % kRing);
    __syncwarp();
    const int cn = c + kRing - 1;
    w_issue(W, cn <= c1 ? cn : -1, cn % kRing);
  }
  __pipeline_wait_prior(0);
}

// f(c, slot) for tiles c = c1 .. c0 (descending).
template <class F>
__device__ __forceinline__ void w_tiles_down(const WarpCtx &W, int c1, int c0, F &&f) {
  if (c1 < c0) return;
#pragma unroll
  for (int k = 0; k < kRing - 1; ++k) w_issue(W, c1 - k >= c0 ? c1 - k : -1, (c1 - k + 64 * kRing) % kRing);
  for (int c = c1; c >= c0; --c) {
    __pipeline_wait_prior(kRing - 2);
    __syncwarp();
    f(c, c % kRing);
    __syncwarp();
    const int cn = c - (kRing - 1);
    w_issue(W, cn >= c0 ? cn : -1, (cn + 64 * kRing) % kRing);
  }
  __pipeline_wait_prior(0);
}

__device__ __forceinline__ Row w_row(const WarpCtx &W, int slot, int k) {
  const double2 a = W.sm->rDL[slot][k][W.seg], b = W.sm->rLD[slot][k];
  Row r; r.D = a.x; r.LLD = a.y; r.LD = b.x; r.LD2 = b.y;
  return r;
}

__device__ __forceinline__ int warp_max(int v) {
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min(int v) {
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// The forward state before row r and the backward state at row r, replayed
// from the checkpoints of r's segment (forward: rows c*kTR .. r-1; backward:
// rows top-1 .. r from the state at the segment's top) -- the operations the
// sweeps did, so the values equal the sweeps' at r.
__device__ __forceinline__ void w_states_at(const WarpCtx &W, double lam, int r, Fwd &Fr, Bwd &Br) {
  const int nb = W.nb;
  const int cr = r / kTR, top = min(cr * kTR + kTR, nb - 1);
  const FwdCk fk = W.fck[(int64_t)cr * W.ck_stride + W.tix];
  const BwdCk bk = W.bck[(int64_t)cr * W.ck_stride + W.tix];
  Fr = Fwd{fk.p, fk.q, fk.H, fk.neg};
  for (int i = cr * kTR; i < r; ++i) {
    const double2 dl = __ldg(&W.DL[i]), lv = __ldg(&W.LDv[i]);
    Row R; R.D = dl.x; R.LLD = dl.y; R.LD = lv.x; R.LD2 = lv.y;
    Fr.step_r(R, lam, (i & 7) == 7);
  }
  Br = Bwd{bk.a, bk.b, bk.K, bk.neg};
  for (int i = top - 1; i >= r; --i) {
    const double2 dl = __ldg(&W.DL[i]), lv = __ldg(&W.LDv[i]);
    Row R; R.D = dl.x; R.LLD = dl.y; R.LD = lv.x; R.LD2 = lv.y;
    Br.step_r(R, lam, (i & 7) == 0);
  }
}

// ---------------------------------------------------------------------------
// PAIR execution.  A CTA holds one work item (up to 32 eigenpairs of one node)
// and two warps: warp F (role 0) runs every stationary (top-down) sweep and
// warp B (role 1) every progressive (bottom-up) one, at the same time.  The
// two halves of a twisted factorization are independent until the twist, so
// each factorization costs one sweep of latency instead of two: the full
// factorization (both sweeps, then the twist search split between the warps
// over the segments, each replaying both states from the checkpoints), every
// fixed-twist RQC factorization (rows < r on F, rows > r on B) and the z
// solve (left part on F, right part on B).  The warps meet at CTA barriers
// to exchange the twist quantities; both then run the same RQC control
// (identical inputs, identical decisions); only F writes the side effects.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void put_bck(const WarpCtx &W, int c, const Bwd &B) {
  BwdCk bk; bk.a = B.a; bk.b = B.b; bk.K = B.K; bk.neg = B.neg; bk.pad = 0;
  W.bck[(int64_t)c * W.ck_stride + W.tix] = bk;
}

// Best twist of a range of rows: |gamma| = |N| / |q b| compared by
// cross-multiplication; among equal values the lowest row (the full search
// scans downward and keeps a later row on ties).
struct TwistPart {
  double N, den;
  int r, have;
};

// Per-CTA exchange between the two warps (per lane).
struct PairX {
  double fp[32], fq[32], fH[32];
  double ba[32], bb[32], bK[32];
  int fneg[32], bneg[32], ok[2][32];
  double eN[2][32], eden[2][32];
  int er[2][32], ehave[2][32];
};

// Twist search over segments c = chi .. clo (descending), replaying the
// forward state of each segment from its checkpoint into shared memory and
// the backward state from its checkpoint (both sweeps of the same
// factorization wrote them).
__device__ __forceinline__ TwistPart w_eval_segments(const WarpCtx &W, double lam, int chi, int clo) {
  const int nb = W.nb, L = W.lane;
  WarpSmem &S = *W.sm;
  TwistPart T;
  T.N = 0; T.den = 0; T.r = nb - 1; T.have = 0;
  if (chi < clo) return T;
  FwdCk ckn = W.fck[(int64_t)chi * W.ck_stride + W.tix];
  BwdCk bkn = W.bck[(int64_t)chi * W.ck_stride + W.tix];
  bool have = false;
  w_tiles_down(W, chi, clo, [&](int c, int slot) {
    const int r0 = c * kTR, r1 = min(r0 + kTR, nb);
    const FwdCk ck = ckn;
    const BwdCk bk = bkn;
    if (c > clo) {
      ckn = W.fck[(int64_t)(c - 1) * W.ck_stride + W.tix];
      bkn = W.bck[(int64_t)(c - 1) * W.ck_stride + W.tix];
    }
    Fwd G{ck.p, ck.q, ck.H, 0};
    Bwd B{bk.a, bk.b, bk.K, bk.neg};
    // only (N, den, r) are tracked; the rest is recomputed at r (w_states_at)
    auto eval = [&](int k) {
      const double fpi = S.sA[k][L], fqi = S.sB[k][L];
      const double qb = fqi * B.b;
      const double N = fma(fpi, B.b, fma(B.a, fqi, lam * qb));
      const bool better = (!have || (fabs(N) * fabs(T.den) <= fabs(T.N) * fabs(qb))) && qb != 0.0 &&
                          isfinite(N);
      have |= better;
      T.r = better ? r0 + k : T.r;
      T.N = better ? N : T.N;
      T.den = better ? qb : T.den;
    };
    if (r1 < nb) {  // full segment, rows r0 .. r0+15 all below nb-1
#pragma unroll 8
      for (int k = 0; k < kTR; ++k) {
        S.sA[k][L] = G.p; S.sB[k][L] = G.q;
        G.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
      }
#pragma unroll 8
      for (int k = kTR - 1; k >= 0; --k) {
        B.step_r(w_row(W, slot, k), lam, (k & 7) == 0);
        eval(k);
      }
    } else {  // the top segment: rows r0 .. nb-1
      const int nr = r1 - r0;
      for (int k = 0; k < nr; ++k) {
        S.sA[k][L] = G.p; S.sB[k][L] = G.q;
        if (k < nr - 1) G.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
      }
      eval(nr - 1);
      for (int k = nr - 2; k >= 0; --k) {
        B.step_r(w_row(W, slot, k), lam, (k & 7) == 0);
        eval(k);
      }
    }
    return false;
  });
  T.have = have;
  return T;
}

// Full twisted factorization of every lane at its own lambda (inactive lanes
// compute too, on a harmless shift; their results are ignored).  Called by
// both warps of the pair.
__device__ __forceinline__ Twist w_full_pair(const WarpCtx &W, double lam, int role, PairX &X) {
  const int nb = W.nb, L = W.lane;
  bool ok;
  if (role == 0) {  // stationary sweep, checkpoints of every segment
    Fwd F{-lam, 1.0, 0.0, 0};
    w_tiles_up(W, 0, W.nseg - 1, [&](int c, int slot) {
      put_fck(VecCtx{nullptr, nullptr, nb, W.nseg, W.fck, W.bck, W.ck_stride}, c, W.tix, F);
      const int r0 = c * kTR;
      const int rows = min(kTR, nb - 1 - r0);  // rows carrying LLD
      if (rows == kTR) {
#pragma unroll
        for (int k = 0; k < kTR; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
      } else {
        for (int k = 0; k < rows; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
      }
      return false;
    });
    ok = isfinite(F.p) && isfinite(F.q);
  } else {  // progressive sweep, checkpoint = state at row min(r0 + kTR, nb - 1)
    Bwd B{__ldg(&W.DL[nb - 1]).x - lam, 1.0, 0.0, 0};
    w_tiles_down(W, W.nseg - 1, 0, [&](int c, int slot) {
      put_bck(W, c, B);
      const int r0 = c * kTR, r1 = min(r0 + kTR, nb);
      if (r1 < nb) {
#pragma unroll
        for (int k = kTR - 1; k >= 0; --k) B.step_r(w_row(W, slot, k), lam, (k & 7) == 0);
      } else {
        for (int k = r1 - r0 - 2; k >= 0; --k) B.step_r(w_row(W, slot, k), lam, (k & 7) == 0);
      }
      return false;
    });
    ok = isfinite(B.a) && isfinite(B.b);
  }
  __syncthreads();  // both sweeps' checkpoints are written (global memory, CTA scope)
  // twist search: F takes the lower half of the segments, B the upper half
  const int h = W.nseg / 2;
  const TwistPart T = role == 0 ? w_eval_segments(W, lam, h - 1, 0) : w_eval_segments(W, lam, W.nseg - 1, h);
  X.eN[role][L] = T.N; X.eden[role][L] = T.den; X.er[role][L] = T.r;
  X.ehave[role][L] = T.have; X.ok[role][L] = ok;
  __syncthreads();
  // combine: the lower half wins ties (it comes later in the downward scan)
  const bool h0 = X.ehave[0][L], h1 = X.ehave[1][L];
  const bool low = h0 && (!h1 || fabs(X.eN[0][L]) * fabs(X.eden[1][L]) <= fabs(X.eN[1][L]) * fabs(X.eden[0][L]));
  const int s = low ? 0 : 1;
  const double bN = X.eN[s][L], bden = X.eden[s][L];
  Twist tw;
  tw.r = X.er[s][L];
  Fwd Fr;
  Bwd Br;
  w_states_at(W, lam, tw.r, Fr, Br);  // both warps: the same values
  tw.gamma = bN / bden;
  tw.nrm2 = 1.0 + Fr.H / (Fr.q * Fr.q) + Br.K / (Br.b * Br.b);
  tw.negc = Fr.neg + Br.neg + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = X.ok[0][L] && X.ok[1][L] && (h0 || h1) && isfinite(tw.gamma) && isfinite(tw.nrm2);
  __syncthreads();  // X is reused by the next exchange
  return tw;
}

// One tile of a fixed-twist factorization's forward part: rows r0 .. r0+15
// below the lane's rf.  A lane whose rf lies beyond the tile steps all 16
// rows unpredicated (the common case: one branch per TILE, not per row -- a
// per-row predicate compiled to a reconvergence block per row, ~40 % of the
// vector kernels' stall samples); the lane whose rf falls inside the tile
// steps the rest in a loop; lanes past rf do nothing.
__device__ __forceinline__ void w_fixed_fwd_tile(const WarpCtx &W, int slot, int r0, int rf, double lam, Fwd &F) {
  auto fstep = [&](int k) {
    const Row R = w_row(W, slot, k);
    const double t = fma(R.D, F.q, F.p);
    F.neg += negbit(t, F.q);
    F.H = R.LD2 * fma(F.q, F.q, F.H);
    F.p = fma(-lam, t, R.LLD * F.p);
    F.q = t;
    if ((k & 7) == 7) fwd_rescale(F.p, F.q, F.H);
  };
  if (r0 + kTR <= rf) {
#pragma unroll
    for (int k = 0; k < kTR; ++k) fstep(k);
  } else if (r0 < rf) {
    for (int k = 0; k < rf - r0; ++k) fstep(k);
  }
}
// The backward part's tile: rows top .. r0 (descending) at or above the
// lane's rb and below nb - 1.
__device__ __forceinline__ void w_fixed_bwd_tile(const WarpCtx &W, int slot, int r0, int top, int rb, double lam,
                                                 Bwd &B) {
  auto bstep = [&](int k) {
    const Row R = w_row(W, slot, k);
    const double u = fma(R.LLD, B.b, B.a);
    B.neg += negbit(u, B.b);
    B.K = R.LD2 * fma(B.b, B.b, B.K);
    B.a = fma(-lam, u, R.D * B.a);
    B.b = u;
    if ((k & 7) == 0) bwd_rescale(B.a, B.b, B.K);
  };
  const int nb = W.nb;
  if (top - r0 + 1 == kTR && top < nb - 1) {
    if (r0 >= rb) {
#pragma unroll
      for (int k = kTR - 1; k >= 0; --k) bstep(k);
    } else if (r0 + kTR > rb) {
      for (int k = kTR - 1; k >= rb - r0; --k) bstep(k);
    }
  } else {
    for (int k = top - r0; k >= 0; --k) {
      const int i = r0 + k;
      if (i < nb - 1 && i >= rb) bstep(k);
    }
  }
}

// Fixed-twist factorization of every lane at its own (lambda, r): F steps
// rows 0..r-1 (ascending tiles up to the warp's largest r), B rows nb-2..r
// (descending tiles down to the smallest r), each lane only its own rows.
// Checkpoints: F of the segments below r, B of the segments from r / kTR
// (the solve replays them).  Called by both warps of the pair.
__device__ __forceinline__ Twist w_fixed_pair(const WarpCtx &W, double lam, int r, bool active, int role,
                                              PairX &X) {
  const int nb = W.nb, L = W.lane;
  if (role == 0) {
    Fwd F{-lam, 1.0, 0.0, 0};
    const int rf = active ? r : 0;  // an idle lane steps no rows
    const VecCtx Xc{nullptr, nullptr, nb, W.nseg, W.fck, W.bck, W.ck_stride};
    const int cf = warp_max(rf > 0 ? (rf - 1) / kTR : -1);
    w_tiles_up(W, 0, cf, [&](int c, int slot) {
      const int r0 = c * kTR;
      if (r0 < rf) put_fck(Xc, c, W.tix, F);
      w_fixed_fwd_tile(W, slot, r0, rf, lam, F);
      return false;
    });
    X.fp[L] = F.p; X.fq[L] = F.q; X.fH[L] = F.H; X.fneg[L] = F.neg;
  } else {
    Bwd B{__ldg(&W.DL[nb - 1]).x - lam, 1.0, 0.0, 0};
    const int rb = active ? r : nb - 1;  // backward steps into rows [rb, nb - 1)
    const int cb = warp_min(rb / kTR);
    w_tiles_down(W, W.nseg - 1, cb, [&](int c, int slot) {
      const int r0 = c * kTR;
      const int top = min(r0 + kTR, nb) - 1;  // rows r0 .. top in this tile
      if (c >= rb / kTR) put_bck(W, c, B);    // state at row min(r0 + kTR, nb - 1)
      w_fixed_bwd_tile(W, slot, r0, top, rb, lam, B);
      return false;
    });
    X.ba[L] = B.a; X.bb[L] = B.b; X.bK[L] = B.K; X.bneg[L] = B.neg;
  }
  __syncthreads();
  const double Fp = X.fp[L], Fq = X.fq[L], FH = X.fH[L];
  const double Ba = X.ba[L], Bb = X.bb[L], BK = X.bK[L];
  const double qb = Fq * Bb;
  const double N = fma(Fp, Bb, fma(Ba, Fq, lam * qb));
  Twist tw;
  tw.r = r;
  tw.gamma = N / qb;
  tw.nrm2 = 1.0 + FH / (Fq * Fq) + BK / (Bb * Bb);
  tw.negc = X.fneg[L] + X.bneg[L] + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = isfinite(tw.gamma) && isfinite(tw.nrm2) && qb != 0.0;
  __syncthreads();
  return tw;
}

// Each lane writes its chunk rows [a, b] (values sA[0 .. b-a][lane]) to its
// own column: 16-byte stores when the chunk start is 16-byte aligned.
__device__ __forceinline__ void w_flush(const WarpCtx &W, int a, int b, double *col) {
  const int L = W.lane;
  if (b < a) return;
  double *dst = col + a;
  const int cnt = b - a + 1;
  if ((((uintptr_t)dst) & 15) == 0) {
    int k = 0;
    for (; k + 1 < cnt; k += 2) {
      double2 v = make_double2(W.sm->sA[k][L], W.sm->sA[k + 1][L]);
      __stcg(reinterpret_cast<double2 *>(dst + k), v);
    }
    if (k < cnt) __stcg(dst + k, W.sm->sA[k][L]);
  } else {
    for (int k = 0; k < cnt; ++k) __stcg(dst + k, W.sm->sA[k][L]);
  }
}

// ---------------------------------------------------------------------------
// SINGLE-warp execution (one warp per item, both sweeps in sequence): fewer
// resources per item, used for the pieces that overlap the tree levels.
// ---------------------------------------------------------------------------

// Full twisted factorization of every lane at its own lambda (inactive lanes
// compute too, on a harmless shift; their results are ignored).
__device__ __forceinline__ Twist w_twist_full(const WarpCtx &W, double lam) {
  const int nb = W.nb, L = W.lane;
  WarpSmem &S = *W.sm;
  // ---- forward (stationary) sweep with checkpoints
  Fwd F{-lam, 1.0, 0.0, 0};
  w_tiles_up(W, 0, W.nseg - 1, [&](int c, int slot) {
    put_fck(VecCtx{nullptr, nullptr, nb, W.nseg, W.fck, W.bck, W.ck_stride}, c, W.tix, F);
    const int r0 = c * kTR;
    const int rows = min(kTR, nb - 1 - r0);  // rows carrying LLD
    if (rows == kTR) {
#pragma unroll
      for (int k = 0; k < kTR; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
    } else {
      for (int k = 0; k < rows; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
    }
    return false;
  });
  bool ok = isfinite(F.p) && isfinite(F.q);
  // ---- backward (progressive) sweep with replay and argmin |gamma|
  Bwd B{__ldg(&W.DL[nb - 1]).x - lam, 1.0, 0.0, 0};
  int best_r = nb - 1;
  double bN = 0, bden = 0;
  bool have = false;
  FwdCk ckn = W.fck[(int64_t)(W.nseg - 1) * W.ck_stride + W.tix];
  w_tiles_down(W, W.nseg - 1, 0, [&](int c, int slot) {
    const int r0 = c * kTR, r1 = min(r0 + kTR, nb);
    {
      BwdCk bk; bk.a = B.a; bk.b = B.b; bk.K = B.K; bk.neg = B.neg; bk.pad = 0;  // state at row min(r0 + kTR, nb - 1)
      W.bck[(int64_t)c * W.ck_stride + W.tix] = bk;
    }
    const FwdCk ck = ckn;
    if (c > 0) ckn = W.fck[(int64_t)(c - 1) * W.ck_stride + W.tix];
    Fwd G{ck.p, ck.q, 0.0, 0};
    // the replay needs (p, q) only: the step and rescale of Fwd without H
    // and the negcount (the same p, q values: the rescale factor depends on
    // p and q alone)
    auto gstep = [&](const Row &R, bool rescale) {
      const double t = fma(R.D, G.q, G.p);
      G.p = fma(-lam, t, R.LLD * G.p);
      G.q = t;
      if (rescale) {
        const double f = pow2_scale(min(max_exp(G.p, G.q), 2045));
        G.p *= f; G.q *= f;
      }
    };
    // argmin |gamma| by cross-multiplication, branch-free (selects) so that
    // the next rows' progressive steps are scheduled across the comparison;
    // only (N, den, r) are tracked -- the partial norms and negcounts at the
    // chosen r are recomputed after the sweep from the two checkpoints
    auto eval = [&](int k) {
      const double fpi = S.sA[k][L], fqi = S.sB[k][L];
      const double qb = fqi * B.b;
      const double N = fma(fpi, B.b, fma(B.a, fqi, lam * qb));
      const bool better = (!have || (fabs(N) * fabs(bden) <= fabs(bN) * fabs(qb))) && qb != 0.0 &&
                          isfinite(N);
      have |= better;
      best_r = better ? r0 + k : best_r;
      bN = better ? N : bN;
      bden = better ? qb : bden;
    };
    if (r1 < nb) {  // full segment, rows r0 .. r0+15 all below nb-1
#pragma unroll 8
      for (int k = 0; k < kTR; ++k) {
        S.sA[k][L] = G.p; S.sB[k][L] = G.q;
        gstep(w_row(W, slot, k), (k & 7) == 7);
      }
#pragma unroll 8
      for (int k = kTR - 1; k >= 0; --k) {
        B.step_r(w_row(W, slot, k), lam, (k & 7) == 0);
        eval(k);
      }
    } else {  // the top segment: rows r0 .. nb-1
      const int nr = r1 - r0;
      for (int k = 0; k < nr; ++k) {
        S.sA[k][L] = G.p; S.sB[k][L] = G.q;
        if (k < nr - 1) gstep(w_row(W, slot, k), (k & 7) == 7);
      }
      eval(nr - 1);
      for (int k = nr - 2; k >= 0; --k) {
        B.step_r(w_row(W, slot, k), lam, (k & 7) == 0);
        eval(k);
      }
    }
    return false;
  });
  ok &= isfinite(B.a) && isfinite(B.b) && have;
  // the partial norms and negcounts at r from the checkpoints
  Fwd Fr;
  Bwd Br;
  w_states_at(W, lam, best_r, Fr, Br);
  Twist tw;
  tw.r = best_r;
  tw.gamma = bN / bden;
  tw.nrm2 = 1.0 + Fr.H / (Fr.q * Fr.q) + Br.K / (Br.b * Br.b);
  tw.negc = Fr.neg + Br.neg + ((tw.gamma < 0.0) ? 1 : 0);
  tw.ok = ok && isfinite(tw.gamma) && isfinite(tw.nrm2);
  return tw;
}

// Fixed-twist factorization of every lane at its own (lambda, r): forward
// rows 0..r-1 (ascending tiles up to the warp's largest r) and backward rows
// nb-2..r (descending tiles down to the smallest r), each lane stepping only
// its own rows.  No argmin, no replay: one pass of simple steps per
// direction.
__device__ __forceinline__ Twist w_twist_fixed(const WarpCtx &W, double lam, int r, bool active) {
  const int nb = W.nb;
  Fwd F{-lam, 1.0, 0.0, 0};
  Bwd B{__ldg(&W.DL[nb - 1]).x - lam, 1.0, 0.0, 0};
  // an idle lane steps no rows and does not widen the warp's tile ranges
  const int rf = active ? r : 0;        // forward rows [0, rf)
  const int rb = active ? r : nb - 1;   // backward steps into rows [rb, nb - 1)
  const VecCtx X{nullptr, nullptr, nb, W.nseg, W.fck, W.bck, W.ck_stride};
  // ---- forward: tiles 0 .. (max r - 1) / kTR; checkpoints of the segments
  // below r (the replayed solve reads them)
  const int cf = warp_max(rf > 0 ? (rf - 1) / kTR : -1);
  w_tiles_up(W, 0, cf, [&](int c, int slot) {
    const int r0 = c * kTR;
    if (r0 < rf) put_fck(X, c, W.tix, F);
    w_fixed_fwd_tile(W, slot, r0, rf, lam, F);
    return false;
  });
  // ---- backward: tiles nseg-1 .. r / kTR
  const int cb = warp_min(rb / kTR);
  w_tiles_down(W, W.nseg - 1, cb, [&](int c, int slot) {
    const int r0 = c * kTR;
    const int top = min(r0 + kTR, nb) - 1;  // rows r0 .. top in this tile
    if (c >= rb / kTR) {
      BwdCk bk; bk.a = B.a; bk.b = B.b;    // state at row min(r0 + kTR, nb - 1)
      W.bck[(int64_t)c * W.ck_stride + W.tix] = bk;
    }
    w_fixed_bwd_tile(W, slot, r0, top, rb, lam, B);
    return false;
  });
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

// z pass of every active lane: z_r = 1, written as scale * z to col[0 .. nb),
// DIVISION-FREE ("projective z").  Left of r the solve is
// z_i = -LD_i (q_i / t_i) z_{i+1}; the replay stores q_{i+1} = t_i f_i (f_i
// the exact power-of-two rescale applied after row i, 1 elsewhere), so with
// y_i = z_i / q_i:   y_i = -LD_i f_i y_{i+1},  z_i = y_i q_i,  y_r = 1 / q_r.
// Right of r, z_{i+1} = -LD_i (b_{i+1} / u_{i+1}) z_i with b_i = u_{i+1} f_i,
// so with v_i = z_i / b_i:   v_{i+1} = -LD_i f_i v_i,  z_{i+1} = v_{i+1} b_{i+1},
// v_r = 1 / b_r.  Two multiplications per row, no reciprocal, and a zero
// pivot (t_i = 0, so q_{i+1} = 0) needs no special case: z_{i+1} = 0 and
// z_i = -(LD_{i+1} / LD_i) z_{i+2} follow from the recurrences (the
// zero-component rule of O10 step 4, reached without evaluating it).
__device__ __forceinline__ void w_solve_left(const WarpCtx &W, double lam, int r, double scale, double *col,
                                             bool active) {
  const int L = W.lane;
  WarpSmem &S = *W.sm;
  if (active) col[r] = scale;
  // rows i < r, descending segments
  const int clast = (active && r > 0) ? (r - 1) / kTR : -1;
  const int cmax = warp_max(clast);
  double y = 0.0;
  FwdCk ckn = W.fck[(int64_t)max(min(clast, cmax), 0) * W.ck_stride + W.tix];
  w_tiles_down(W, cmax, 0, [&](int c, int slot) {
    const bool on = c <= clast;
    const int r0 = c * kTR, r1 = on ? min(r0 + kTR, r) : r0;  // rows [r0, r1)
    const FwdCk ck = ckn;
    if (on && c > 0) ckn = W.fck[(int64_t)(c - 1) * W.ck_stride + W.tix];
    double p = ck.p, q = ck.q;
    auto rep = [&](int k) {  // state before row r0 + k -> before r0 + k + 1
      const Row R = w_row(W, slot, k);
      S.sA[k][L] = q;  // q_i
      const double t = fma(R.D, q, p);
      p = fma(-lam, t, R.LLD * p);
      q = t;
      double f = 1.0;
      if ((k & 7) == 7) {
        f = pow2_scale(min(max_exp(p, q), 2045));
        p *= f; q *= f;
      }
      S.sC[k][L] = -R.LD * f;
    };
    if (on && r1 == r0 + kTR) {
#pragma unroll
      for (int k = 0; k < kTR; ++k) rep(k);
    } else if (on) {
      for (int k = 0; k < r1 - r0; ++k) rep(k);
    }
    if (on && r1 == r) y = scale / q;  // y_r = z_r / q_r (q_r != 0: the twist's |gamma_r| is finite)
    auto zstep = [&](int k) {
      y *= S.sC[k][L];
      const double zi = y * S.sA[k][L];
      S.sA[k][L] = (fabs(zi) >= kTiny) ? zi : 0.0;  // reading 17
    };
    if (r1 - r0 == kTR) {
#pragma unroll
      for (int k = kTR - 1; k >= 0; --k) zstep(k);
    } else {
      for (int k = r1 - r0 - 1; k >= 0; --k) zstep(k);
    }
    w_flush(W, r0, r1 - 1, col);  // chunk rows r0 .. r1-1 from sA[0 ..]
    return false;
  });
}

__device__ __forceinline__ void w_solve_right(const WarpCtx &W, double lam, int r, double scale, double *col,
                                              bool active) {
  const int nb = W.nb, L = W.lane;
  WarpSmem &S = *W.sm;
  // rows i > r, ascending segments
  const int cfirst = (active && r < nb - 1) ? r / kTR : W.nseg;
  const int cmin = warp_min(cfirst);
  double v = 0.0;
  BwdCk bkn = W.bck[(int64_t)min(max(cfirst, cmin), W.nseg - 1) * W.ck_stride + W.tix];
  w_tiles_up(W, cmin, W.nseg - 1, [&](int c, int slot) {
    const bool on = c >= cfirst;
    const int r0 = c * kTR;
    const int top = min(r0 + kTR, nb - 1);   // checkpoint row
    const int lo_i = on ? max(r0, r) : top;  // rows i in [lo_i, top) give z_{i+1}
    const BwdCk bk = bkn;
    if (on && c + 1 < W.nseg) bkn = W.bck[(int64_t)(c + 1) * W.ck_stride + W.tix];
    double a = bk.a, b = bk.b;
    auto rep = [&](int k) {  // state at row r0 + k + 1 -> at row r0 + k
      const Row R = w_row(W, slot, k);
      S.sA[k][L] = b;  // b_{i+1}
      const double u = fma(R.LLD, b, a);
      a = fma(-lam, u, R.D * a);
      b = u;
      double f = 1.0;
      if ((k & 7) == 0) {
        f = pow2_scale(min(max_exp(a, b), 2045));
        a *= f; b *= f;
      }
      S.sC[k][L] = -R.LD * f;
    };
    if (on && lo_i == r0 && top == r0 + kTR) {
#pragma unroll
      for (int k = kTR - 1; k >= 0; --k) rep(k);
    } else if (on) {
      for (int k = top - 1 - r0; k >= lo_i - r0; --k) rep(k);
    }
    if (on && lo_i == r) v = scale / b;  // v_r = z_r / b_r
    // z_{i+1} for i in [lo_i, top): chunk rows lo_i+1 .. top, stored at sA[i - lo_i]
    // (ascending i: index i - lo_i <= i - r0 was already read)
    auto ystep = [&](int k, int o) {
      v *= S.sC[k][L];
      const double zn = v * S.sA[k][L];
      S.sA[o][L] = (fabs(zn) >= kTiny) ? zn : 0.0;
    };
    if (lo_i == r0 && top == r0 + kTR) {
#pragma unroll
      for (int k = 0; k < kTR; ++k) ystep(k, k);
    } else {
      for (int i = lo_i; i < top; ++i) ystep(i - r0, i - lo_i);
    }
    w_flush(W, lo_i + 1, top, col);
    return false;
  });
}

__device__ __forceinline__ void w_twist_solve(const WarpCtx &W, double lam, int r, double scale, double *col,
                                              bool active) {
  w_solve_left(W, lam, r, scale, col, active);
  w_solve_right(W, lam, r, scale, col, active);
}

// The pair's solve: F the rows below r (and r itself), B the rows above.
__device__ __forceinline__ void w_solve_pair(const WarpCtx &W, double lam, int r, double scale, double *col,
                                             bool active, int role) {
  if (role == 0) w_solve_left(W, lam, r, scale, col, active);
  else w_solve_right(W, lam, r, scale, col, active);
}

// Reading 24 (amended): the shift after an RQ step `delta` from `lam` in the
// bracket [lo, hi].  A step that leaves the bracket by at most 4 eps |lam +
// delta| is a rounding-level overshoot of an eigenvalue that sits at the
// bracket's end: the end itself.  Otherwise a step leaving the bracket from
// the interior is clamped to the violated end and one from an end bisects;
// after those safeguard steps `delta_prev` is reset, because the next
// correction is compared (reading 10's stagnation test) with a step that was
// not taken -- a bisection halves it by construction, and the test then
// stopped a linearly converging lane far from the eigenvalue (zero-diagonal
// T, eigenvalue 0 at a bracket end: tests/test_gpu_edge.py).  `stuck`: the
// bracket is two adjacent doubles (converged).
__device__ __forceinline__ double rqc_next(double lam, double delta, double lo, double hi, double &delta_prev,
                                           bool &stuck) {
  stuck = false;
  double nw = lam + delta;
  delta_prev = delta;
  if (nw <= lo || nw >= hi) {
    const double slack = 4.0 * kEps * fabs(nw);
    if (nw <= lo && lo - nw <= slack) {
      nw = lo;
    } else if (nw >= hi && nw - hi <= slack) {
      nw = hi;
    } else if (lam == lo || lam == hi) {
      nw = 0.5 * (lo + hi);
      delta_prev = CUDART_INF;
      if (nw <= lo || nw >= hi) stuck = true;
    } else {
      nw = (nw <= lo) ? lo : hi;
      delta_prev = CUDART_INF;
    }
  }
  return nw;
}

// One work item: up to 32 tasks of one node.
struct WarpItem {
  int32_t node;    // node of the first task (the item's tasks may span up to kMaxSeg nodes of one block)
  int32_t t0, t1;  // task ids [t0, t1) (tasks of one node are consecutive)
  int32_t nsegs;   // nodes in the item (host bookkeeping)
};

struct WVecArgs {
  const Node *nodes;
  const double2 *LDv;        // global (LD, LD^2) per row
  const VecTask *tasks;
  const int *task_list;      // optional: item task indices go through this list
  const WarpItem *items;
  int nitems;
  double *lo, *hi;           // slot brackets (node coordinates)
  const int *slot_j;         // block-local 1-based eigen index per slot
  FwdCk *fck;
  BwdCk *bck;
  int64_t ck_stride;         // >= number of tasks + 32 (columns ntask + lane: idle lanes)
  int ntask;
  double *Z; int64_t ldz;    // modes 0, 2: Z columns (tk.col), node rows at N.row0
  double *lam_out;           // modes 0, 2: final lambda (node coordinates) per task
  int mode;                  // 0: RQC (reading 10); 2: one factorization at the bracket
                             // midpoint (RQC fallback); 3, 4: the split RQC's phases
                             // (k_wvectors_split)
  int rqc_max;               // mode 0: factorizations before the fallback
  int *fail_list;            // mode 0: tasks that did not converge (appended as task_base + tix)
  int *fail_count;
  int task_base;             // global index of this launch's task 0
  unsigned long long *ctr;   // [0] factorizations, [1] fallbacks, [2..3] nudges, [4..7] slowest item
  unsigned long long *hist;  // mode 0 / 4: eigenpairs by twisted factorizations of their RQC ([k], k = min(count, 15))
  struct RqcState *state;    // modes 3, 4: per-task RQC state between the split phases
  int *rkey;                 // mode 3: per-task twist index (sort key)
};

// An eigenpair's RQC is done after `nfact` twisted factorizations: the call's
// total and the histogram (mrrr_get_rqc_histogram).
__device__ __forceinline__ void rqc_count(const WVecArgs &A, unsigned long long nfact) {
  atomicAdd(&A.ctr[0], nfact);
  if (A.hist) atomicAdd(&A.hist[nfact < 15ull ? nfact : 15ull], 1ull);
}

constexpr int kPairThreads = 64;  // pair kernel: one item per CTA, warp F + warp B
constexpr int kSingleWarps = 2;   // single-warp kernel: independent items per CTA

__device__ __forceinline__ void wvec_pair_body(const WVecArgs &A) {
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  const int role = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  if (item >= A.nitems) return;  // whole CTA
  const WarpItem It = A.items[item];
  const bool active = It.t0 + lane < It.t1;
  const int pos = active ? It.t0 + lane : It.t1 - 1;  // idle lanes: the item's last task
  const int tix = A.task_list ? A.task_list[pos] : pos;
  const VecTask tk = A.tasks[tix];
  const Node N = A.nodes[tk.node];  // this lane's node (the item's nodes share one block)
  WarpCtx W;
  W.DL = N.DL; W.LDv = A.LDv + N.row0; W.nb = N.nb; W.nseg = (N.nb + kTR - 1) / kTR;
  W.lane = lane;
  W.sm = reinterpret_cast<WarpSmem *>(wsm_raw) + role;
  w_segments(W, A.tasks[pos].node, active);  // position order: nodes unchanged by task_list
  PairX &X = *reinterpret_cast<PairX *>(wsm_raw + 2 * sizeof(WarpSmem));
  W.fck = A.fck; W.bck = A.bck; W.ck_stride = A.ck_stride;
  const int64_t spare = A.ntask + lane;   // idle lanes checkpoint into spare columns
  W.tix = active ? tix : spare;
  const bool lead = role == 0;            // side effects by warp F only
  double lo = A.lo[tk.slot], hi = A.hi[tk.slot];
  if (N.nb == 1) {
    if (active && lead) { A.Z[tk.col * A.ldz + N.row0] = 1.0; A.lam_out[tix] = __ldg(&N.DL[0]).x; }
    return;
  }
  double lam = (A.mode == 2 || isnan(tk.lam0)) ? 0.5 * (lo + hi) : tk.lam0;
  unsigned long long nfact = 0;
  Twist tw;
  const long long clk0 = clock64();
  // full factorization; nudge lambda if not finite (overflow insurance, reading 25)
  {
    double nudge = 2.0 * kEps * fabs(lam) + kTiny;
    const double lam_base = lam;
    for (int tries = 0; tries < 60; ++tries) {
      tw = w_full_pair(W, lam, role, X);
      ++nfact;
      if (g_force_nudge && tries == 0) tw.ok = false;  // diagnostic (MRRR_FORCE_NUDGE)
      if (!__any_sync(0xffffffffu, active && !tw.ok)) break;
      if (active && !tw.ok) {
        lam = lam_base + nudge; nudge *= 2.0;
        if (lead) {
          atomicAdd(&A.ctr[2], 1ull);
          if (A.ctr[3] == 0)  // first failure: record why (debug aid, MRRR_TRACE)
            A.ctr[3] = 1 + (isfinite(tw.gamma) ? 0 : 2) + (isfinite(tw.nrm2) ? 0 : 4);
        }
      }
    }
  }
  double lam_fin = lam;
  const long long clk_full = clock64();
  if (A.mode == 0) {
    // O10 RQC (readings 10, 24): stop when |delta| <= 4 eps |lambda| or
    // fl(lambda + delta) == lambda; a step leaving [lo, hi] from the interior
    // is clamped to the violated end, from an end it bisects.  A lane that
    // has converged keeps its factorization (its checkpoint column is parked
    // on a spare column while the other lanes iterate).
    const int j = A.slot_j[tk.slot];
    bool conv = !active, failed = false;
    Twist best = tw;
    const int best_r0 = tw.r;
    double lam_best = lam, delta_prev = CUDART_INF;
    for (int it = 1;; ++it) {
      if (!conv) {
        if (tw.negc >= j) { if (lam < hi) hi = lam; } else { if (lam > lo) lo = lam; }
        const double delta = tw.gamma / tw.nrm2;
        if (g_debug_rqc && (blockDim.x != kPairThreads || threadIdx.x < 32))
          printf("rqc task %d it %d lam %.17g r %d gamma %.6g nrm2 %.6g delta %.6g negc %d j %d lo %.17g hi %.17g\n",
                 tix, it, lam, tw.r, tw.gamma, tw.nrm2, delta, tw.negc, j, lo, hi);
        // stop (reading 10): |delta| <= 4 eps |lambda|, fl(lambda + delta) ==
        // lambda, or stagnation (the correction no longer halves)
        if (fabs(delta) <= 4.0 * kEps * fabs(lam) || lam + delta == lam ||
            (it > 1 && (fabs(delta) >= 0.5 * fabs(delta_prev) || fabs(delta_prev) <= g_rqc_prev_tol * fabs(lam)))) {
          conv = true; best = tw; lam_best = lam; lam_fin = lam + delta;
        } else {
          bool stuck;
          const double nw = rqc_next(lam, delta, lo, hi, delta_prev, stuck);
          if (stuck) { conv = true; best = tw; lam_best = lam; lam_fin = lam; }          lam = nw;
        }
        if (!conv && it >= A.rqc_max) { conv = true; failed = true; }
        if (conv) W.tix = spare;  // park: later factorizations must not touch its checkpoints
      }
      if (__all_sync(0xffffffffu, conv)) break;
      // later iterations keep the first factorization's twist index
      tw = w_fixed_pair(W, lam, best_r0, !conv, role, X);
      if (!conv) ++nfact;
      if (!conv && !tw.ok) { conv = true; failed = true; W.tix = spare; }
    }
    const long long clk_rqc = clock64();
    W.tix = active ? tix : spare;
    tw = best;
    lam = lam_best;
    if (active && failed && lead) {
      // O10 fallback, deferred: the bracket goes back to the slot; the host
      // refines it to 4 eps and a mode-2 pass writes the vector
      A.lo[tk.slot] = lo; A.hi[tk.slot] = hi;
      A.fail_list[atomicAdd(A.fail_count, 1)] = A.task_base + tix;
      atomicAdd(&A.ctr[1], 1ull);
    }
    // failed lanes skip the solve (their column is written by the fallback)
    const double sc = 1.0 / sqrt(tw.nrm2);
    w_solve_pair(W, lam, tw.r, sc, A.Z + tk.col * A.ldz + N.row0, active && !failed, role);
    if (lead) {
      if (active && !failed) A.lam_out[tix] = lam_fin;
      if (active) rqc_count(A, nfact);
      if (lane == 0) {  // slowest item: cycles of the first factorization, the RQC loop, the solve;
                        // factorizations of the item (MRRR_TRACE)
        const long long clk_end = clock64();
        atomicMax(&A.ctr[4], (unsigned long long)(clk_full - clk0));
        atomicMax(&A.ctr[5], (unsigned long long)(clk_rqc - clk_full));
        atomicMax(&A.ctr[6], (unsigned long long)(clk_end - clk_rqc));
        atomicMax(&A.ctr[7], nfact);
      }
    }
    return;
  }
  // mode 2: the vector of the one factorization at the refined midpoint
  const double sc = 1.0 / sqrt(tw.nrm2);
  w_solve_pair(W, lam, tw.r, sc, A.Z + tk.col * A.ldz + N.row0, active, role);
  if (active && lead) {
    A.lam_out[tix] = lam_fin;
    atomicAdd(&A.ctr[0], nfact);
  }
}

__device__ __forceinline__ void wvec_single_body(const WVecArgs &A) {
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kSingleWarps + wid;
  if (item >= A.nitems) return;  // whole warp
  const WarpItem It = A.items[item];
  const bool active = It.t0 + lane < It.t1;
  const int pos = active ? It.t0 + lane : It.t1 - 1;  // idle lanes: the item's last task
  const int tix = A.task_list ? A.task_list[pos] : pos;
  const VecTask tk = A.tasks[tix];
  const Node N = A.nodes[tk.node];  // this lane's node (the item's nodes share one block)
  WarpCtx W;
  W.DL = N.DL; W.LDv = A.LDv + N.row0; W.nb = N.nb; W.nseg = (N.nb + kTR - 1) / kTR;
  W.lane = lane;
  W.sm = reinterpret_cast<WarpSmem *>(wsm_raw) + wid;
  w_segments(W, A.tasks[pos].node, active);  // position order: nodes unchanged by task_list
  W.fck = A.fck; W.bck = A.bck; W.ck_stride = A.ck_stride;
  const int64_t spare = A.ntask + lane;   // idle lanes checkpoint into spare columns
  W.tix = active ? tix : spare;
  double lo = A.lo[tk.slot], hi = A.hi[tk.slot];
  if (N.nb == 1) {
    if (active) { A.Z[tk.col * A.ldz + N.row0] = 1.0; A.lam_out[tix] = __ldg(&N.DL[0]).x; }
    return;
  }
  double lam = (A.mode == 2 || isnan(tk.lam0)) ? 0.5 * (lo + hi) : tk.lam0;
  unsigned long long nfact = 0;
  Twist tw;
  const long long clk0 = clock64();
  // full factorization; nudge lambda if not finite (overflow insurance, reading 25)
  {
    double nudge = 2.0 * kEps * fabs(lam) + kTiny;
    const double lam_base = lam;
    for (int tries = 0; tries < 60; ++tries) {
      tw = w_twist_full(W, lam);
      ++nfact;
      if (g_force_nudge && tries == 0) tw.ok = false;  // diagnostic (MRRR_FORCE_NUDGE)
      if (!__any_sync(0xffffffffu, active && !tw.ok)) break;
      if (active && !tw.ok) {
        lam = lam_base + nudge; nudge *= 2.0;
        atomicAdd(&A.ctr[2], 1ull);
        if (A.ctr[3] == 0) {  // first failure: record why (debug aid, MRRR_TRACE)
          A.ctr[3] = 1 + (isfinite(tw.gamma) ? 0 : 2) + (isfinite(tw.nrm2) ? 0 : 4);
        }
      }
    }
  }
  double lam_fin = lam;
  const long long clk_full = clock64();
  if (A.mode == 0) {
    // O10 RQC (readings 10, 24): stop when |delta| <= 4 eps |lambda| or
    // fl(lambda + delta) == lambda; a step leaving [lo, hi] from the interior
    // is clamped to the violated end, from an end it bisects.  A lane that
    // has converged keeps its factorization (its checkpoint column is parked
    // on a spare column while the other lanes iterate).
    const int j = A.slot_j[tk.slot];
    bool conv = !active, failed = false;
    Twist best = tw;
    const int best_r0 = tw.r;
    double lam_best = lam, delta_prev = CUDART_INF;
    for (int it = 1;; ++it) {
      if (!conv) {
        if (tw.negc >= j) { if (lam < hi) hi = lam; } else { if (lam > lo) lo = lam; }
        const double delta = tw.gamma / tw.nrm2;
        if (g_debug_rqc && (blockDim.x != kPairThreads || threadIdx.x < 32))
          printf("rqc task %d it %d lam %.17g r %d gamma %.6g nrm2 %.6g delta %.6g negc %d j %d lo %.17g hi %.17g\n",
                 tix, it, lam, tw.r, tw.gamma, tw.nrm2, delta, tw.negc, j, lo, hi);
        // stop (reading 10): |delta| <= 4 eps |lambda|, fl(lambda + delta) ==
        // lambda, or stagnation (the correction no longer halves)
        if (fabs(delta) <= 4.0 * kEps * fabs(lam) || lam + delta == lam ||
            (it > 1 && (fabs(delta) >= 0.5 * fabs(delta_prev) || fabs(delta_prev) <= g_rqc_prev_tol * fabs(lam)))) {
          conv = true; best = tw; lam_best = lam; lam_fin = lam + delta;
        } else {
          bool stuck;
          const double nw = rqc_next(lam, delta, lo, hi, delta_prev, stuck);
          if (stuck) { conv = true; best = tw; lam_best = lam; lam_fin = lam; }          lam = nw;
        }
        if (!conv && it >= A.rqc_max) { conv = true; failed = true; }
        if (conv) W.tix = spare;  // park: later factorizations must not touch its checkpoints
      }
      if (__all_sync(0xffffffffu, conv)) break;
      // later iterations keep the first factorization's twist index
      tw = w_twist_fixed(W, lam, best_r0, !conv);
      if (!conv) ++nfact;
      if (!conv && !tw.ok) { conv = true; failed = true; W.tix = spare; }
    }
    const long long clk_rqc = clock64();
    W.tix = active ? tix : spare;
    tw = best;
    lam = lam_best;
    if (active && failed) {
      // O10 fallback, deferred: the bracket goes back to the slot; the host
      // refines it to 4 eps and a mode-2 pass writes the vector
      A.lo[tk.slot] = lo; A.hi[tk.slot] = hi;
      A.fail_list[atomicAdd(A.fail_count, 1)] = A.task_base + tix;
      atomicAdd(&A.ctr[1], 1ull);
    }
    // failed lanes skip the solve (their column is written by the fallback)
    const double sc = 1.0 / sqrt(tw.nrm2);
    w_twist_solve(W, lam, tw.r, sc, A.Z + tk.col * A.ldz + N.row0, active && !failed);
    if (active && !failed) A.lam_out[tix] = lam_fin;
    if (active) rqc_count(A, nfact);
    if (lane == 0) {  // slowest warp: cycles of the first factorization, the RQC loop, the solve;
                      // factorizations of the warp (MRRR_TRACE)
      const long long clk_end = clock64();
      atomicMax(&A.ctr[4], (unsigned long long)(clk_full - clk0));
      atomicMax(&A.ctr[5], (unsigned long long)(clk_rqc - clk_full));
      atomicMax(&A.ctr[6], (unsigned long long)(clk_end - clk_rqc));
      atomicMax(&A.ctr[7], nfact);
    }
    return;
  }
  // mode 2: the vector of the one factorization at the refined midpoint
  const double sc = 1.0 / sqrt(tw.nrm2);
  w_twist_solve(W, lam, tw.r, sc, A.Z + tk.col * A.ldz + N.row0, active);
  if (active) {
    A.lam_out[tix] = lam_fin;
    atomicAdd(&A.ctr[0], nfact);
  }
}

// ---------------------------------------------------------------------------
// SPLIT execution of the single-warp kernel.  Lanes of an item are
// consecutive eigenvalues whose twist indices r lie anywhere in the node, so
// a fixed-twist factorization (rows < r forward, rows > r backward) and the
// solve walk the union of the lanes' ranges -- about 2 nb rows per warp
// where each lane needs nb.  Phase 1 (mode 3) runs the full factorization
// and the first RQC update and stores each task's state; the host's stream
// then sorts every node's tasks by r (segmented radix sort); phase 2 (mode 4)
// runs the rest of the RQC and the solve with the items' lanes taken in that
// order (task_list), so the lanes of a warp share one row window.  Per-lane
// arithmetic is unchanged (bit-identical results; the state is stored and
// reloaded exactly).
// ---------------------------------------------------------------------------
struct RqcState {
  double lam, lo, hi, delta_prev, lam_best, lam_fin, gamma, nrm2;
  int r, negc, best_r0, flags;  // flags: 1 converged, 2 failed, 4 twist ok
  unsigned long long nfact;
};

// The RQC update after a factorization `tw` at `lam` (iteration `it`), O10
// readings 10 and 24 (the code of wvec_single_body's loop).
struct RqcLane {
  double lam, lo, hi, delta_prev, lam_best, lam_fin;
  Twist best;
  bool conv, failed;
  __device__ __forceinline__ void update(const Twist &tw, int j, int it, int rqc_max) {
    if (tw.negc >= j) { if (lam < hi) hi = lam; } else { if (lam > lo) lo = lam; }
    const double delta = tw.gamma / tw.nrm2;
    if (fabs(delta) <= 4.0 * kEps * fabs(lam) || lam + delta == lam ||
        (it > 1 && (fabs(delta) >= 0.5 * fabs(delta_prev) || fabs(delta_prev) <= g_rqc_prev_tol * fabs(lam)))) {
      conv = true; best = tw; lam_best = lam; lam_fin = lam + delta;
    } else {
      bool stuck;
      const double nw = rqc_next(lam, delta, lo, hi, delta_prev, stuck);
      if (stuck) { conv = true; best = tw; lam_best = lam; lam_fin = lam; }      lam = nw;
    }
    if (!conv && it >= rqc_max) { conv = true; failed = true; }
  }
};

__device__ __forceinline__ void wvec_split_body(const WVecArgs &A) {
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kSingleWarps + wid;
  if (item >= A.nitems) return;  // whole warp
  const WarpItem It = A.items[item];
  const bool active = It.t0 + lane < It.t1;
  const int pos = active ? It.t0 + lane : It.t1 - 1;  // idle lanes: the item's last task
  const int tix = A.task_list ? A.task_list[pos] : pos;
  const VecTask tk = A.tasks[tix];
  const Node N = A.nodes[tk.node];  // this lane's node (the item's nodes share one block)
  WarpCtx W;
  W.DL = N.DL; W.LDv = A.LDv + N.row0; W.nb = N.nb; W.nseg = (N.nb + kTR - 1) / kTR;
  W.lane = lane;
  W.sm = reinterpret_cast<WarpSmem *>(wsm_raw) + wid;
  w_segments(W, A.tasks[pos].node, active);  // position order: nodes unchanged by task_list
  W.fck = A.fck; W.bck = A.bck; W.ck_stride = A.ck_stride;
  const int64_t spare = A.ntask + lane;
  W.tix = active ? tix : spare;
  const int j = A.slot_j[tk.slot];
  if (A.mode == 3) {
    if (N.nb == 1) return;  // phase 2 writes it
    double lam = isnan(tk.lam0) ? 0.5 * (A.lo[tk.slot] + A.hi[tk.slot]) : tk.lam0;
    unsigned long long nfact = 0;
    Twist tw;
    {
      double nudge = 2.0 * kEps * fabs(lam) + kTiny;
      const double lam_base = lam;
      for (int tries = 0; tries < 60; ++tries) {
        tw = w_twist_full(W, lam);
        ++nfact;
        if (g_force_nudge && tries == 0) tw.ok = false;  // diagnostic (MRRR_FORCE_NUDGE)
        if (!__any_sync(0xffffffffu, active && !tw.ok)) break;
        if (active && !tw.ok) {
          lam = lam_base + nudge; nudge *= 2.0;
          atomicAdd(&A.ctr[2], 1ull);
          if (A.ctr[3] == 0) A.ctr[3] = 1 + (isfinite(tw.gamma) ? 0 : 2) + (isfinite(tw.nrm2) ? 0 : 4);
        }
      }
    }
    RqcLane Q;
    Q.lam = lam; Q.lo = A.lo[tk.slot]; Q.hi = A.hi[tk.slot]; Q.delta_prev = CUDART_INF;
    Q.lam_best = lam; Q.lam_fin = lam; Q.best = tw; Q.conv = !active; Q.failed = false;
    if (!Q.conv) Q.update(tw, j, 1, A.rqc_max);
    if (active) {
      RqcState st;
      st.lam = Q.lam; st.lo = Q.lo; st.hi = Q.hi; st.delta_prev = Q.delta_prev;
      st.lam_best = Q.lam_best; st.lam_fin = Q.lam_fin; st.gamma = Q.best.gamma; st.nrm2 = Q.best.nrm2;
      st.r = Q.best.r; st.negc = Q.best.negc; st.best_r0 = tw.r;
      st.flags = (Q.conv ? 1 : 0) | (Q.failed ? 2 : 0) | (Q.best.ok ? 4 : 0);
      st.nfact = nfact;
      A.state[tix] = st;
      A.rkey[tix] = tw.r;
    }
    return;
  }
  // ---- mode 4: the rest of the RQC and the solve, lanes in twist order
  if (N.nb == 1) {
    if (active) { A.Z[tk.col * A.ldz + N.row0] = 1.0; A.lam_out[tix] = __ldg(&N.DL[0]).x; }
    return;
  }
  RqcLane Q;
  int best_r0 = 0;
  unsigned long long nfact = 0;
  if (active) {
    const RqcState st = A.state[tix];
    Q.lam = st.lam; Q.lo = st.lo; Q.hi = st.hi; Q.delta_prev = st.delta_prev;
    Q.lam_best = st.lam_best; Q.lam_fin = st.lam_fin;
    Q.best.r = st.r; Q.best.gamma = st.gamma; Q.best.nrm2 = st.nrm2; Q.best.negc = st.negc;
    Q.best.ok = (st.flags & 4) != 0;
    Q.conv = (st.flags & 1) != 0; Q.failed = (st.flags & 2) != 0;
    best_r0 = st.best_r0; nfact = st.nfact;
  } else {
    Q.lam = 0.0; Q.lo = 0.0; Q.hi = 0.0; Q.delta_prev = CUDART_INF; Q.lam_best = 0.0; Q.lam_fin = 0.0;
    Q.best.r = 0; Q.best.gamma = 0.0; Q.best.nrm2 = 1.0; Q.best.negc = 0; Q.best.ok = true;
    Q.conv = true; Q.failed = false;
  }
  // Phase 2 checkpoints go to the lane's POSITION column (consecutive within
  // the item: coalesced), not the task's (scattered by the twist sort).  A
  // lane whose RQC converged in phase 1 rebuilds its checkpoints there with
  // one fixed-twist factorization at (lam_best, r): the same recurrences over
  // the same rows as the full factorization's, so the same values (bit for
  // bit); phase-1 columns are never read here.
  W.tix = active ? pos : spare;
  {
    const bool refac = active && Q.conv && !Q.failed;
    if (__any_sync(0xffffffffu, refac)) {
      (void)w_twist_fixed(W, Q.lam_best, Q.best.r, refac);
      if (refac) ++nfact;
    }
  }
  if (Q.conv) W.tix = spare;  // parked: its column holds its converged factorization
  for (int it = 1;;) {
    if (__all_sync(0xffffffffu, Q.conv)) break;
    const Twist tw = w_twist_fixed(W, Q.lam, best_r0, !Q.conv);
    if (!Q.conv) ++nfact;
    ++it;
    if (!Q.conv && !tw.ok) { Q.conv = true; Q.failed = true; }
    else if (!Q.conv) Q.update(tw, j, it, A.rqc_max);
    if (Q.conv) W.tix = spare;
  }
  W.tix = active ? pos : spare;
  if (active && Q.failed) {
    A.lo[tk.slot] = Q.lo; A.hi[tk.slot] = Q.hi;
    A.fail_list[atomicAdd(A.fail_count, 1)] = A.task_base + tix;
    atomicAdd(&A.ctr[1], 1ull);
  }
  const double sc = 1.0 / sqrt(Q.best.nrm2);
  w_twist_solve(W, Q.lam_best, Q.best.r, sc, A.Z + tk.col * A.ldz + N.row0, active && !Q.failed);
  if (active && !Q.failed) A.lam_out[tix] = Q.lam_fin;
  if (active) rqc_count(A, nfact);
  if (lane == 0) atomicMax(&A.ctr[7], nfact);
}

// The split RQC on warp PAIRS (round 2): mode 3 = the full factorization
// (w_full_pair, nudges as in wvec_pair_body) and the first RQC update, state
// stored per task; the host sorts each node's tasks by twist index; mode 4 =
// the remaining fixed-twist factorizations (w_fixed_pair) and the solve
// (w_solve_pair) with the item's lanes in that order.  After the regrouping
// the lanes of an item share one row window, so warp F's forward rows
// (below the largest r of the item) and warp B's backward rows (above the
// smallest r) no longer both span the node.  Per-lane arithmetic is
// wvec_pair_body's / wvec_split_body's (bit-identical results).
__device__ __forceinline__ void wvec_pair_split_body(const WVecArgs &A) {
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  const int role = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  if (item >= A.nitems) return;  // whole CTA
  const WarpItem It = A.items[item];
  const bool active = It.t0 + lane < It.t1;
  const int pos = active ? It.t0 + lane : It.t1 - 1;
  const int tix = A.task_list ? A.task_list[pos] : pos;
  const VecTask tk = A.tasks[tix];
  const Node N = A.nodes[tk.node];
  WarpCtx W;
  W.DL = N.DL; W.LDv = A.LDv + N.row0; W.nb = N.nb; W.nseg = (N.nb + kTR - 1) / kTR;
  W.lane = lane;
  W.sm = reinterpret_cast<WarpSmem *>(wsm_raw) + role;
  w_segments(W, A.tasks[pos].node, active);
  PairX &X = *reinterpret_cast<PairX *>(wsm_raw + 2 * sizeof(WarpSmem));
  W.fck = A.fck; W.bck = A.bck; W.ck_stride = A.ck_stride;
  const int64_t spare = A.ntask + lane;
  W.tix = active ? tix : spare;
  const bool lead = role == 0;
  const int j = A.slot_j[tk.slot];
  if (A.mode == 3) {
    if (N.nb == 1) return;  // phase 2 writes it
    double lam = isnan(tk.lam0) ? 0.5 * (A.lo[tk.slot] + A.hi[tk.slot]) : tk.lam0;
    unsigned long long nfact = 0;
    Twist tw;
    {
      double nudge = 2.0 * kEps * fabs(lam) + kTiny;
      const double lam_base = lam;
      for (int tries = 0; tries < 60; ++tries) {
        tw = w_full_pair(W, lam, role, X);
        ++nfact;
        if (g_force_nudge && tries == 0) tw.ok = false;  // diagnostic (MRRR_FORCE_NUDGE)
        if (!__any_sync(0xffffffffu, active && !tw.ok)) break;
        if (active && !tw.ok) {
          lam = lam_base + nudge; nudge *= 2.0;
          if (lead) {
            atomicAdd(&A.ctr[2], 1ull);
            if (A.ctr[3] == 0) A.ctr[3] = 1 + (isfinite(tw.gamma) ? 0 : 2) + (isfinite(tw.nrm2) ? 0 : 4);
          }
        }
      }
    }
    RqcLane Q;
    Q.lam = lam; Q.lo = A.lo[tk.slot]; Q.hi = A.hi[tk.slot]; Q.delta_prev = CUDART_INF;
    Q.lam_best = lam; Q.lam_fin = lam; Q.best = tw; Q.conv = !active; Q.failed = false;
    if (!Q.conv) Q.update(tw, j, 1, A.rqc_max);
    if (active && lead) {
      RqcState st;
      st.lam = Q.lam; st.lo = Q.lo; st.hi = Q.hi; st.delta_prev = Q.delta_prev;
      st.lam_best = Q.lam_best; st.lam_fin = Q.lam_fin; st.gamma = Q.best.gamma; st.nrm2 = Q.best.nrm2;
      st.r = Q.best.r; st.negc = Q.best.negc; st.best_r0 = tw.r;
      st.flags = (Q.conv ? 1 : 0) | (Q.failed ? 2 : 0) | (Q.best.ok ? 4 : 0);
      st.nfact = nfact;
      A.state[tix] = st;
      A.rkey[tix] = tw.r;
    }
    return;
  }
  // ---- mode 4: the rest of the RQC and the solve, lanes in twist order
  if (N.nb == 1) {
    if (active && lead) { A.Z[tk.col * A.ldz + N.row0] = 1.0; A.lam_out[tix] = __ldg(&N.DL[0]).x; }
    return;
  }
  RqcLane Q;
  int best_r0 = 0;
  unsigned long long nfact = 0;
  if (active) {
    const RqcState st = A.state[tix];
    Q.lam = st.lam; Q.lo = st.lo; Q.hi = st.hi; Q.delta_prev = st.delta_prev;
    Q.lam_best = st.lam_best; Q.lam_fin = st.lam_fin;
    Q.best.r = st.r; Q.best.gamma = st.gamma; Q.best.nrm2 = st.nrm2; Q.best.negc = st.negc;
    Q.best.ok = (st.flags & 4) != 0;
    Q.conv = (st.flags & 1) != 0; Q.failed = (st.flags & 2) != 0;
    best_r0 = st.best_r0; nfact = st.nfact;
  } else {
    Q.lam = 0.0; Q.lo = 0.0; Q.hi = 0.0; Q.delta_prev = CUDART_INF; Q.lam_best = 0.0; Q.lam_fin = 0.0;
    Q.best.r = 0; Q.best.gamma = 0.0; Q.best.nrm2 = 1.0; Q.best.negc = 0; Q.best.ok = true;
    Q.conv = true; Q.failed = false;
  }
  // checkpoints in the lane's POSITION column (wvec_split_body); a lane that
  // converged in phase 1 rebuilds them with one fixed-twist factorization
  W.tix = active ? pos : spare;
  {
    const bool refac = active && Q.conv && !Q.failed;
    if (__any_sync(0xffffffffu, refac)) {
      (void)w_fixed_pair(W, Q.lam_best, Q.best.r, refac, role, X);
      if (refac) ++nfact;
    }
  }
  if (Q.conv) W.tix = spare;
  for (int it = 1;;) {
    if (__all_sync(0xffffffffu, Q.conv)) break;
    const Twist tw = w_fixed_pair(W, Q.lam, best_r0, !Q.conv, role, X);
    if (!Q.conv) ++nfact;
    ++it;
    if (!Q.conv && !tw.ok) { Q.conv = true; Q.failed = true; }
    else if (!Q.conv) Q.update(tw, j, it, A.rqc_max);
    if (Q.conv) W.tix = spare;
  }
  W.tix = active ? pos : spare;
  if (active && Q.failed && lead) {
    A.lo[tk.slot] = Q.lo; A.hi[tk.slot] = Q.hi;
    A.fail_list[atomicAdd(A.fail_count, 1)] = A.task_base + tix;
    atomicAdd(&A.ctr[1], 1ull);
  }
  const double sc = 1.0 / sqrt(Q.best.nrm2);
  w_solve_pair(W, Q.lam_best, Q.best.r, sc, A.Z + tk.col * A.ldz + N.row0, active && !Q.failed, role);
  if (lead) {
    if (active && !Q.failed) A.lam_out[tix] = Q.lam_fin;
    if (active) rqc_count(A, nfact);
    if (lane == 0) atomicMax(&A.ctr[7], nfact);
  }
}

// At most 168 registers per thread (6 CTAs of 64 threads per SM by
// registers): the vector pieces share the SMs with the tree's kernels.
__global__ void __launch_bounds__(32 * kSingleWarps, 6) k_wvectors_split(WVecArgs A) { wvec_split_body(A); }

__global__ void __launch_bounds__(kPairThreads, 6) k_wvectors_pair(WVecArgs A) { wvec_pair_body(A); }
__global__ void __launch_bounds__(kPairThreads, 6) k_wvectors_psplit(WVecArgs A) { wvec_pair_split_body(A); }
__global__ void __launch_bounds__(32 * kSingleWarps, 6) k_wvectors(WVecArgs A) { wvec_single_body(A); }

}  // namespace mrrr
