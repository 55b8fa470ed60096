// Microbenchmark (test tooling): cycles per row of the refinement sweep of
// k_refine_warp (projective Sturm steps, rows through a cp.async ring of
// 16-row tiles, rescale every 8 rows, sign-change count), one warp per CTA,
// one shift per lane, against variants that drop one ingredient each.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1205_2107_b200/csrc
//      tools/ubench_sturm.cu -o tools/ubench_sturm
#include <cuda_pipeline.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace mrrr;

constexpr int kT = 16, kRing = 6;

// VAR: 0 as k_refine_warp<1>; 1 no count; 2 no rescale; 3 rows from registers
// (no ring); 4 rescale every 16; 5 two shifts per lane; 6 count via predicate
// popc-free add (t < 0) != (q < 0) on doubles; 7 rescale test folded (frexp-free
// exponent of q only)
template <int VAR>
__global__ void k_sweep(const double2 *DL, int nb, double mu0, double *out, long long *cyc) {
  __shared__ double2 ring[kRing][kT];
  const int lane = threadIdx.x;
  const double mu = mu0 * (1.0 + 1e-3 * (lane + 32 * blockIdx.x));
  const double mu2 = mu * (1.0 + 1e-6);
  Sturm st, st2;
  sturm_init(st, mu);
  sturm_init(st2, mu2);
  st2.c = 0;
  const int body = nb - 1, ntile = (body + kT - 1) / kT;
  auto issue = [&](int t) {
    const int row = t * kT + lane;
    if (lane < kT && t < ntile && row < body) __pipeline_memcpy_async(&ring[t % kRing][lane], &DL[row], sizeof(double2));
    __pipeline_commit();
  };
  double2 rv[kT];
  if (VAR == 3 || VAR == 10)
    for (int k = 0; k < kT; ++k) rv[k] = DL[k];
  bool ok = true;
  __syncwarp();
  const long long c0 = clock64();
  if (VAR != 3 && VAR != 10)
#pragma unroll
    for (int k = 0; k < kRing - 1; ++k) issue(k);
  for (int t = 0; t < ntile; ++t) {
    double2 v[kT];
    unsigned xs[kT];
    unsigned sbits = (unsigned)hi32(st.q) >> 31;  // sign of q before the tile
    if (VAR != 3 && VAR != 10) {
      __pipeline_wait_prior(kRing - 2);
      __syncwarp();
      const double2 *T = ring[t % kRing];
#pragma unroll
      for (int k = 0; k < kT; ++k) v[k] = T[k];
      if (VAR == 11 || VAR == 12) asm volatile("" ::: "memory");
    } else {
#pragma unroll
      for (int k = 0; k < kT; ++k) v[k] = rv[k];
    }
#pragma unroll
    for (int k = 0; k < kT; ++k) {
      if (VAR == 1) {
        const double tt = fma(v[k].x, st.q, st.p);
        st.p = fma(-mu, tt, v[k].y * st.p);
        st.q = tt;
      } else if (VAR == 14) {
        const double tt = fma(v[k].x, st.q, st.p);
        sbits = __funnelshift_l((unsigned)hi32(tt), sbits, 1);  // sign bit of t enters at bit 0
        st.p = fma(-mu, tt, v[k].y * st.p);
        st.q = tt;
      } else if (VAR == 13) {
        const double tt = fma(v[k].x, st.q, st.p);
        if (k & 1) st2.c += negbit(tt, st.q); else st.c += negbit(tt, st.q);
        st.p = fma(-mu, tt, v[k].y * st.p);
        st.q = tt;
      } else if (VAR == 8 || VAR == 9 || VAR == 10 || VAR == 12) {
        const double tt = fma(v[k].x, st.q, st.p);
        xs[k] = (unsigned)(hi32(tt) ^ hi32(st.q));
        st.p = fma(-mu, tt, v[k].y * st.p);
        st.q = tt;
      } else if (VAR == 6) {
        const double tt = fma(v[k].x, st.q, st.p);
        st.c += ((tt < 0.0) != (st.q < 0.0));
        st.p = fma(-mu, tt, v[k].y * st.p);
        st.q = tt;
      } else {
        sturm_step(st, v[k].x, v[k].y, mu);
        if (VAR == 5) sturm_step(st2, v[k].x, v[k].y, mu2);
      }
      if (VAR != 2 && ((VAR == 4 || VAR == 9) ? (k == kT - 1) : ((k & 7) == 7))) {
        if (VAR == 7) {
          const int e = (hi32(st.q) >> 20) & 0x7ff;
          const double f = pow2_scale(min(e, 2045));
          st.p *= f; st.q *= f;
          ok &= e < 2047;
        } else {
          ok &= sturm_rescale(st);
          if (VAR == 5) ok &= sturm_rescale(st2);
        }
      }
    }
    if (VAR == 14) {  // sign changes between consecutive bits 0..16
      st.c += __popc((sbits ^ (sbits >> 1)) & 0xffffu);
    }
    if (VAR == 8 || VAR == 9 || VAR == 10 || VAR == 12) {
      unsigned a = 0;
#pragma unroll
      for (int k = 0; k < kT; ++k) a += xs[k] >> 31;
      st.c += a;
    }
    if (VAR != 3 && VAR != 10) {
      __syncwarp();
      issue(t + kRing - 1);
    }
  }
  if (VAR != 3 && VAR != 10) __pipeline_wait_prior(0);
  const long long c1 = clock64();
  out[blockIdx.x * 32 + lane] = st.p + st.q + st.c + (ok ? 0 : 1) + (VAR == 5 ? st2.q + st2.c : 0.0) +
                                 (VAR == 13 ? st2.c : 0.0);
  if (lane == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int VAR>
void run(const double2 *dDL, int nb, double *dout, long long *dcyc, int grid, const char *name) {
  k_sweep<VAR><<<grid, 32>>>(dDL, nb, 0.3, dout, dcyc);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_sweep<VAR><<<grid, 32>>>(dDL, nb, 0.3, dout, dcyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<long long> c(grid);
  cudaMemcpy(c.data(), dcyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (long long x : c) avg += (double)x;
  avg /= grid;
  std::vector<double> o(grid * 32);
  cudaMemcpy(o.data(), dout, grid * 32 * sizeof(double), cudaMemcpyDeviceToHost);
  double cs = 0;
  for (double x : o) cs += x;
  printf("{\"var\": %d, \"name\": \"%s\", \"grid\": %d, \"cycles_per_row\": %.2f, \"ms\": %.3f, \"checksum\": %.17g}\n",
         VAR, name, grid, avg / (nb - 1), ms, cs);
}


// Tile-size variants of VAR 0 (rows per ring tile TT, lanes copy TT/32 rows each)
template <int TT>
__global__ void k_sweep_tt(const double2 *DL, int nb, double mu0, double *out, long long *cyc) {
  __shared__ double2 ring[kRing][TT];
  const int lane = threadIdx.x;
  const double mu = mu0 * (1.0 + 1e-3 * (lane + 32 * blockIdx.x));
  Sturm st;
  sturm_init(st, mu);
  const int body = nb - 1, ntile = (body + TT - 1) / TT;
  auto issue = [&](int t) {
    for (int r = lane; r < TT; r += 32) {
      const int row = t * TT + r;
      if (t < ntile && row < body) __pipeline_memcpy_async(&ring[t % kRing][r], &DL[row], sizeof(double2));
    }
    __pipeline_commit();
  };
  bool ok = true;
  __syncwarp();
  const long long c0 = clock64();
#pragma unroll
  for (int k = 0; k < kRing - 1; ++k) issue(k);
  for (int t = 0; t < ntile; ++t) {
    __pipeline_wait_prior(kRing - 2);
    __syncwarp();
    const double2 *T = ring[t % kRing];
#pragma unroll
    for (int k = 0; k < TT; ++k) {
      const double2 v = T[k];
      sturm_step(st, v.x, v.y, mu);
      if ((k & 7) == 7) ok &= sturm_rescale(st);
    }
    __syncwarp();
    issue(t + kRing - 1);
  }
  __pipeline_wait_prior(0);
  const long long c1 = clock64();
  out[blockIdx.x * 32 + lane] = st.p + st.q + st.c + (ok ? 0 : 1);
  if (lane == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int TT>
void run_tt(const double2 *dDL, int nb, double *dout, long long *dcyc, int grid) {
  k_sweep_tt<TT><<<grid, 32>>>(dDL, nb, 0.3, dout, dcyc);
  cudaDeviceSynchronize();
  k_sweep_tt<TT><<<grid, 32>>>(dDL, nb, 0.3, dout, dcyc);
  cudaDeviceSynchronize();
  std::vector<long long> c(grid);
  cudaMemcpy(c.data(), dcyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (long long x : c) avg += (double)x;
  std::vector<double> o(grid * 32);
  cudaMemcpy(o.data(), dout, grid * 32 * sizeof(double), cudaMemcpyDeviceToHost);
  double cs = 0;
  for (double x : o) cs += x;
  printf("{\"tile_rows\": %d, \"grid\": %d, \"cycles_per_row\": %.2f, \"checksum\": %.17g}\n", TT, grid,
         avg / grid / (nb - 1), cs);
}

int main() {
  const int nb = 20000;
  std::vector<double2> h(nb);
  srand(7);
  for (int i = 0; i < nb; ++i) {
    const double D = 0.5 + (double)rand() / RAND_MAX, L = 0.3 * ((double)rand() / RAND_MAX - 0.5);
    h[i] = make_double2(D, L * L * D);
  }
  double2 *dDL;
  double *dout;
  long long *dcyc;
  cudaMalloc(&dDL, nb * sizeof(double2));
  cudaMalloc(&dout, 148 * 16 * 32 * sizeof(double));
  cudaMalloc(&dcyc, 148 * 16 * sizeof(long long));
  cudaMemcpy(dDL, h.data(), nb * sizeof(double2), cudaMemcpyHostToDevice);
  for (int grid : {148, 148 * 4, 148 * 16}) {
    run<0>(dDL, nb, dout, dcyc, grid, "as k_refine_warp<1>");
    run<1>(dDL, nb, dout, dcyc, grid, "no count");
    run<2>(dDL, nb, dout, dcyc, grid, "no rescale");
    run<3>(dDL, nb, dout, dcyc, grid, "rows in registers");
    run<4>(dDL, nb, dout, dcyc, grid, "rescale every 16");
    run<5>(dDL, nb, dout, dcyc, grid, "two shifts per lane");
    run<6>(dDL, nb, dout, dcyc, grid, "count by compare");
    run<7>(dDL, nb, dout, dcyc, grid, "rescale on q exponent");
    run<8>(dDL, nb, dout, dcyc, grid, "count summed per tile");
    run<9>(dDL, nb, dout, dcyc, grid, "count per tile, rescale every 16");
    run<10>(dDL, nb, dout, dcyc, grid, "count per tile, rows in registers");
    run<11>(dDL, nb, dout, dcyc, grid, "tile loads before the chain");
    run<12>(dDL, nb, dout, dcyc, grid, "tile loads before the chain, count per tile");
    run<13>(dDL, nb, dout, dcyc, grid, "two count accumulators");
    run<14>(dDL, nb, dout, dcyc, grid, "sign bits packed by funnel shift, popc per tile");
  }
  for (int grid : {148, 148 * 16}) {
    run_tt<8>(dDL, nb, dout, dcyc, grid);
    run_tt<16>(dDL, nb, dout, dcyc, grid);
    run_tt<32>(dDL, nb, dout, dcyc, grid);
    run_tt<64>(dDL, nb, dout, dcyc, grid);
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
