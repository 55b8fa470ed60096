// Micro-benchmark (test tooling): one warp, per-row cost of the lockstep
// twisted factorization and solve (kernels_warp.cuh) on a synthetic node.
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_1205_2107_b200/csrc/kernels_warp.cuh"
using namespace mrrr;

__global__ void kb_full(const double2 *DL, const double2 *LDv, int nb, FwdCk *fck, BwdCk *bck, int64_t cs,
                        double *out, int reps) {
  extern __shared__ __align__(16) unsigned char raw[];
  WarpCtx W;
  W.DL = DL; W.LDv = LDv; W.nb = nb; W.nseg = (nb + kTR - 1) / kTR; W.lane = threadIdx.x & 31;
  W.sm = reinterpret_cast<WarpSmem *>(raw); W.fck = fck; W.bck = bck; W.ck_stride = cs; W.tix = W.lane;
  double lam = 0.3 + 1e-3 * W.lane, acc = 0;
  for (int r = 0; r < reps; ++r) { Twist t = w_twist_full(W, lam); acc += t.gamma + t.r; lam += 1e-9; }
  out[W.lane] = acc;
}
__global__ void kb_solve(const double2 *DL, const double2 *LDv, int nb, FwdCk *fck, BwdCk *bck, int64_t cs,
                         double *Z, double *out, int r) {
  extern __shared__ __align__(16) unsigned char raw[];
  WarpCtx W;
  W.DL = DL; W.LDv = LDv; W.nb = nb; W.nseg = (nb + kTR - 1) / kTR; W.lane = threadIdx.x & 31;
  W.sm = reinterpret_cast<WarpSmem *>(raw); W.fck = fck; W.bck = bck; W.ck_stride = cs; W.tix = W.lane;
  double lam = 0.3 + 1e-3 * W.lane;
  w_twist_solve(W, lam, r + W.lane * 7, 1.0, Z + (size_t)W.lane * nb, true);
}


#define SETUP \
  extern __shared__ __align__(16) unsigned char raw[]; \
  WarpCtx W; \
  W.DL = DL; W.LDv = LDv; W.nb = nb; W.nseg = (nb + kTR - 1) / kTR; W.lane = threadIdx.x & 31; \
  W.sm = reinterpret_cast<WarpSmem *>(raw); W.fck = fck; W.bck = bck; W.ck_stride = cs; W.tix = W.lane; \
  double lam = 0.3 + 1e-3 * W.lane;
__global__ void kb_fwd(const double2 *DL, const double2 *LDv, int nb, FwdCk *fck, BwdCk *bck, int64_t cs, double *out) {
  SETUP
  Fwd F{-lam, 1.0, 0.0, 0};
  w_tiles_up(W, 0, W.nseg - 1, [&](int c, int slot) {
    put_fck(VecCtx{nullptr, nullptr, nb, W.nseg, W.fck, W.bck, W.ck_stride}, c, W.tix, F);
    const int rows = min(kTR, nb - 1 - c * kTR);
    if (rows == kTR) {
#pragma unroll
      for (int k = 0; k < kTR; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
    } else {
      for (int k = 0; k < rows; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
    }
    return false;
  });
  out[W.lane] = F.p + F.q + F.H + F.neg;
}
__global__ void kb_fwd_nock(const double2 *DL, const double2 *LDv, int nb, FwdCk *fck, BwdCk *bck, int64_t cs, double *out) {
  SETUP
  Fwd F{-lam, 1.0, 0.0, 0};
  w_tiles_up(W, 0, W.nseg - 1, [&](int c, int slot) {
    const int rows = min(kTR, nb - 1 - c * kTR);
    if (rows == kTR) {
#pragma unroll
      for (int k = 0; k < kTR; ++k) F.step_r(w_row(W, slot, k), lam, (k & 7) == 7);
    }
    return false;
  });
  out[W.lane] = F.p + F.q + F.H + F.neg;
}
__global__ void kb_fwd_plain(const double2 *DL, const double2 *LDv, int nb, FwdCk *fck, BwdCk *bck, int64_t cs, double *out) {
  SETUP
  double p = -lam, q = 1.0;
  w_tiles_up(W, 0, W.nseg - 1, [&](int c, int slot) {
    const int rows = min(kTR, nb - 1 - c * kTR);
    if (rows == kTR) {
#pragma unroll
      for (int k = 0; k < kTR; ++k) {
        const double2 v = W.sm->rDL[slot][k];
        double t = fma(v.x, q, p); p = fma(-lam, t, v.y * p); q = t;
        if ((k & 7) == 7) { int e = max_exp(p, q); double f = pow2_scale(min(e, 2045)); p *= f; q *= f; }
      }
    }
    return false;
  });
  out[W.lane] = p + q;
}

int main() {
  const int n = 20000;
  std::vector<double2> h(n), hl(n);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(0.5, 1.5);
  for (int i = 0; i < n; ++i) { double D = U(g), L = 0.3 * U(g); h[i] = make_double2(D, L * L * D); hl[i] = make_double2(L * D, L * L * D * D); }
  double2 *d, *dl; double *out, *Z; FwdCk *fck; BwdCk *bck;
  int nseg = (n + kTR - 1) / kTR;
  cudaMalloc(&d, n * 16); cudaMalloc(&dl, n * 16); cudaMalloc(&out, 1024); cudaMalloc(&Z, (size_t)32 * n * 8);
  cudaMalloc(&fck, (size_t)nseg * 64 * sizeof(FwdCk)); cudaMalloc(&bck, (size_t)nseg * 64 * sizeof(BwdCk));
  cudaMemcpy(d, h.data(), n * 16, cudaMemcpyHostToDevice); cudaMemcpy(dl, hl.data(), n * 16, cudaMemcpyHostToDevice);
  size_t sm = sizeof(WarpSmem);
  cudaFuncSetAttribute(kb_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(kb_fwd_nock, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(kb_fwd_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(kb_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(kb_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto T = [&](const char *name, auto fn, double passes) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-22s %8.3f ms  %7.1f cyc/row@1.965GHz\n", name, ms, ms * 1e6 / (n * passes) * 1.965);
  };
  T("fwd plain (tiles)", [&] { kb_fwd_plain<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, out); }, 1);
  T("fwd Fwd.step nock", [&] { kb_fwd_nock<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, out); }, 1);
  T("fwd Fwd.step + ck", [&] { kb_fwd<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, out); }, 1);
  T("full x1 (1 warp)", [&] { kb_full<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, out, 1); }, 1);
  T("full x4 (1 warp)", [&] { kb_full<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, out, 4); }, 4);
  T("solve r=n/2", [&] { kb_solve<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, Z, out, n / 2); }, 1);
  T("solve r=100", [&] { kb_solve<<<1, 32, sm>>>(d, dl, n, fck, bck, 64, Z, out, 100); }, 1);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
