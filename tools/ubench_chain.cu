// Micro-benchmark (test tooling): per-row latency of one-thread sweeps.
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_1205_2107_b200/csrc/kernels_tree.cuh"
#include <cuda_pipeline.h>
using namespace mrrr;

__global__ void v_nostore(const double2 *DL, int nb, double sg, double *out) {
  double p = -sg, q = 1.0;
  for (int i = 0; i < nb - 1; ++i) {
    double2 v = __ldg(&DL[i]);
    double t = fma(v.x, q, p);
    p = fma(-sg, t, v.y * p);
    q = t;
    if ((i & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
  }
  out[0] = p; out[1] = q;
}
__global__ void v_stream(const double2 *DL, int nb, double sg, double *out) {
  double p = -sg, q = 1.0;
  stream_rows<8>(DL, 0, nb - 1, [&](int i, const double2 &v) {
    double t = fma(v.x, q, p);
    p = fma(-sg, t, v.y * p);
    q = t;
    if ((i & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
  });
  out[0] = p; out[1] = q;
}
__global__ void v_stream_store(const double2 *DL, int nb, double sg, double *tb, int *sb) {
  double p = -sg, q = 1.0;
  stream_rows<8>(DL, 0, nb, [&](int i, const double2 &v) {
    double t = fma(v.x, q, p);
    tb[i] = t;
    int sh = 0;
    if (i < nb - 1) {
      p = fma(-sg, t, v.y * p); q = t;
      if ((i & 7) == 7) { int ee = max_exp(p, q); sh = 1023 - min(max(ee, 1), 2045); double f = pow2(sh); p *= f; q *= f; }
    }
    sb[i] = sh;
  });
}
__global__ void v_regs(int nb, double sg, double *out) {  // no memory at all
  double p = -sg, q = 1.0, D = 1.5, L = 0.25;
  for (int i = 0; i < nb - 1; ++i) {
    double t = fma(D, q, p);
    p = fma(-sg, t, L * p);
    q = t;
    if ((i & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
    D += 1e-9; 
  }
  out[0] = p; out[1] = q;
}
__global__ void v_smem(const double2 *DL, int nb, double sg, double *out) {  // rows from shared memory
  __shared__ double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = DL[i];
  __syncthreads();
  if (threadIdx.x) return;
  double p = -sg, q = 1.0;
  for (int i = 0; i < nb - 1; ++i) {
    double2 v = sm[i & 2047];
    double t = fma(v.x, q, p);
    p = fma(-sg, t, v.y * p);
    q = t;
    if ((i & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
  }
  out[0] = p; out[1] = q;
}


// warp of 32 chains over the same rows
__global__ void w_global(const double2 *DL, int nb, double *Z, int ldz, int store) {
  int l = threadIdx.x;
  double sg = 0.3 + 1e-3 * l, p = -sg, q = 1.0;
  double *col = Z + (size_t)l * ldz;
  stream_rows<8>(DL, 0, nb - 1, [&](int i, const double2 &v) {
    double t = fma(v.x, q, p);
    p = fma(-sg, t, v.y * p);
    q = t;
    if ((i & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
    if (store) col[i] = t;
  });
  if (!store) Z[l] = p + q;
}
// warp-cooperative smem tiles (cp.async, 4-deep ring of 32-row tiles), lockstep
__global__ void w_tiles(const double2 *DL, int nb, double *Z, int ldz, int store) {
  __shared__ double2 ring[4][32];
  int l = threadIdx.x;
  double sg = 0.3 + 1e-3 * l, p = -sg, q = 1.0;
  double *col = Z + (size_t)l * ldz;
  const int body = nb - 1, nt = (body + 31) / 32;
  auto issue = [&](int t) {
    int r = t * 32 + l;
    if (t < nt && r < body) __pipeline_memcpy_async(&ring[t & 3][l], &DL[r], 16);
    __pipeline_commit();
  };
  issue(0); issue(1); issue(2);
  for (int t = 0; t < nt; ++t) {
    __pipeline_wait_prior(2);
    __syncwarp();
    const double2 *T = ring[t & 3];
    int rows = min(32, body - t * 32);
    if (rows == 32) {
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        double2 v = T[k];
        double tt = fma(v.x, q, p);
        p = fma(-sg, tt, v.y * p);
        q = tt;
        if ((k & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
        if (store) col[t * 32 + k] = tt;
      }
    } else {
      for (int k = 0; k < rows; ++k) {
        double2 v = T[k];
        double tt = fma(v.x, q, p);
        p = fma(-sg, tt, v.y * p);
        q = tt;
        if ((k & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
        if (store) col[t * 32 + k] = tt;
      }
    }
    __syncwarp();
    issue(t + 3);
  }
  if (!store) Z[l] = p + q;
}
// staged stores: z for 32 rows kept in smem, then the warp writes each lane's
// 32-row chunk (256 contiguous bytes) cooperatively
__global__ void w_tiles_coal(const double2 *DL, int nb, double *Z, int ldz) {
  __shared__ double2 ring[4][32];
  __shared__ double zt[32][33];
  int l = threadIdx.x;
  double sg = 0.3 + 1e-3 * l, p = -sg, q = 1.0;
  const int body = nb - 1, nt = body / 32;
  auto issue = [&](int t) {
    int r = t * 32 + l;
    if (t < nt) __pipeline_memcpy_async(&ring[t & 3][l], &DL[r], 16);
    __pipeline_commit();
  };
  issue(0); issue(1); issue(2);
  for (int t = 0; t < nt; ++t) {
    __pipeline_wait_prior(2);
    __syncwarp();
    const double2 *T = ring[t & 3];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      double2 v = T[k];
      double tt = fma(v.x, q, p);
      p = fma(-sg, tt, v.y * p);
      q = tt;
      if ((k & 7) == 7) { int ee = max_exp(p, q); double f = pow2_scale(min(ee, 2045)); p *= f; q *= f; }
      zt[l][k] = tt;
    }
    __syncwarp();
    for (int c = 0; c < 32; ++c) Z[(size_t)c * ldz + t * 32 + l] = zt[c][l];
    __syncwarp();
    issue(t + 3);
  }
}

int main() {
  const int n = 20000;
  std::vector<double2> h(n);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(0.5, 1.5);
  for (auto &x : h) x = make_double2(U(g), U(g) * 0.1);
  double2 *d; double *out, *tb; int *sb;
  cudaMalloc(&d, n * sizeof(double2)); cudaMalloc(&out, 64); cudaMalloc(&tb, n * 8); cudaMalloc(&sb, n * 4);
  cudaMemcpy(d, h.data(), n * sizeof(double2), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto T = [&](const char *name, auto fn) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-16s %8.3f ms  %7.1f ns/row  %6.1f cyc/row@1.965GHz\n", name, ms, ms * 1e6 / n, ms * 1e6 / n * 1.965);
  };
  T("regs", [&] { v_regs<<<1, 1>>>(n, 0.3, out); });
  T("smem", [&] { v_smem<<<1, 128>>>(d, n, 0.3, out); });
  T("nostore", [&] { v_nostore<<<1, 1>>>(d, n, 0.3, out); });
  T("stream", [&] { v_stream<<<1, 1>>>(d, n, 0.3, out); });
  T("stream_store", [&] { v_stream_store<<<1, 1>>>(d, n, 0.3, tb, sb); });
  double *Z; cudaMalloc(&Z, (size_t)32 * n * 8);
  T("warp_glob_nost", [&] { w_global<<<1, 32>>>(d, n, Z, n, 0); });
  T("warp_glob_store", [&] { w_global<<<1, 32>>>(d, n, Z, n, 1); });
  T("warp_tile_nost", [&] { w_tiles<<<1, 32>>>(d, n, Z, n, 0); });
  T("warp_tile_store", [&] { w_tiles<<<1, 32>>>(d, n, Z, n, 1); });
  T("warp_tile_coal", [&] { w_tiles_coal<<<1, 32>>>(d, n, Z, n); });
  T("4w/SM glob_st", [&] { w_global<<<148 * 4, 32>>>(d, n, Z, 0, 1); });
  T("4w/SM tile_coal", [&] { w_tiles_coal<<<148 * 4, 32>>>(d, n, Z, 0); });
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
