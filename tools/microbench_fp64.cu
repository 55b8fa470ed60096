// FP64 microbenchmarks for the B200 roofline denominators.
// Measures: DFMA latency / throughput, IEEE DDIV latency / throughput, and the
// per-step latency/throughput of two Sturm-count step forms (qd-with-division,
// projective division-free).  Prints one JSON object.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e_=(x); if(e_!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e_)); return 1;}}while(0)

__global__ void lat_dfma(double* out, long long* cyc, int iters, double a, double b) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = fma(x, a, b); }
  long long t1 = clock64();
  out[1] = x; cyc[0] = t1 - t0;
}
__global__ void lat_ddiv(double* out, long long* cyc, int iters, double a) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = a / x + 0.5; }
  long long t1 = clock64();
  out[1] = x; cyc[0] = t1 - t0;
}
// qd step: D+ = D + S ; c += D+<0 ; S = S/D+ * LLD - mu
__global__ void lat_qd(double* out, long long* cyc, int iters, double D, double LLD, double mu) {
  double S = -mu; int c = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { double dp = D + S; c += (dp < 0); S = fma(S / dp, LLD, -mu); }
  long long t1 = clock64();
  out[1] = S + c; cyc[0] = t1 - t0;
}
// projective step: t = fma(D,q,p); c += sign(t)^sign(q); p = fma(-mu, t, LLD*p); q = t
__global__ void lat_proj(double* out, long long* cyc, int iters, double D, double LLD, double mu) {
  double p = -mu, q = 1.0; unsigned c = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double t = fma(D, q, p);
    c += ((unsigned)(__double2hiint(t) ^ __double2hiint(q))) >> 31;
    p = fma(-mu, t, LLD * p); q = t;
    if ((i & 7) == 7) { int e = (__double2hiint(q) >> 20) & 0x7ff; double s = __hiloint2double((2046 - e) << 20, 0); p *= s; q *= s; }
  }
  long long t1 = clock64();
  out[1] = p + q + c; cyc[0] = t1 - t0;
}

template <int ILP>
__global__ void tput_dfma(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}
template <int ILP>
__global__ void tput_ddiv(double* out, int iters, double a) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = 1.0 + threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = a / x[k] + 0.75;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}
template <int ILP>
__global__ void tput_qd(double* out, int iters, double D, double LLD, double mu0) {
  double S[ILP], mu[ILP]; int c = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { mu[k] = mu0 + 1e-3 * (threadIdx.x + k); S[k] = -mu[k]; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) { double dp = D + S[k]; c += (dp < 0); S[k] = fma(S[k] / dp, LLD, -mu[k]); }
  }
  double s = c;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += S[k];
  if (s == 12345.678) out[0] = s;
}
template <int ILP>
__global__ void tput_proj(double* out, int iters, double D, double LLD, double mu0) {
  double p[ILP], q[ILP], mu[ILP]; unsigned c = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { mu[k] = mu0 + 1e-3 * (threadIdx.x + k); p[k] = -mu[k]; q[k] = 1.0; }
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < ILP; ++k) {
        double t = fma(D, q[k], p[k]);
        c += ((unsigned)(__double2hiint(t) ^ __double2hiint(q[k]))) >> 31;
        p[k] = fma(-mu[k], t, LLD * p[k]); q[k] = t;
      }
    }
#pragma unroll
    for (int k = 0; k < ILP; ++k) { int e = (__double2hiint(q[k]) >> 20) & 0x7ff; double s = __hiloint2double((2046 - e) << 20, 0); p[k] *= s; q[k] *= s; }
  }
  double s = c;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += p[k] + q[k];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* d; long long* cyc; CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&cyc, 64));
  double one = 1.0; CK(cudaMemcpy(d, &one, 8, cudaMemcpyHostToDevice));
  long long h; const int LI = 1 << 16;
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d", p.name, sms, p.clockRate);
  lat_dfma<<<1,1>>>(d, cyc, LI, 0.999999, 1e-9); lat_dfma<<<1,1>>>(d, cyc, LI, 0.999999, 1e-9); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf(",\"dfma_lat_cyc\":%.2f", (double)h / LI);
  lat_ddiv<<<1,1>>>(d, cyc, LI, 0.7); lat_ddiv<<<1,1>>>(d, cyc, LI, 0.7); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf(",\"ddiv_lat_cyc\":%.2f", (double)h / LI);
  lat_qd<<<1,1>>>(d, cyc, LI, 2.0, 0.5, 0.3); lat_qd<<<1,1>>>(d, cyc, LI, 2.0, 0.5, 0.3); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf(",\"qd_step_lat_cyc\":%.2f", (double)h / LI);
  lat_proj<<<1,1>>>(d, cyc, LI, 2.0, 0.5, 0.3); lat_proj<<<1,1>>>(d, cyc, LI, 2.0, 0.5, 0.3); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf(",\"proj_step_lat_cyc\":%.2f", (double)h / LI);

  const int IT = 1 << 14;
  for (int bpsm : {1, 2, 4, 8}) {
    int blocks = sms * bpsm, thr = 256;
    float ms = timeit([&] { tput_dfma<8><<<blocks, thr>>>(d, IT, 0.999999, 1e-9); });
    double ops = (double)blocks * thr * IT * 8;
    printf(",\"dfma_per_s_b%d\":%.4e", bpsm, ops / (ms * 1e-3));
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int blocks = sms * bpsm, thr = 256;
    float ms = timeit([&] { tput_ddiv<4><<<blocks, thr>>>(d, IT / 4, 0.7); });
    double ops = (double)blocks * thr * (IT / 4) * 4;
    printf(",\"ddiv_per_s_b%d\":%.4e", bpsm, ops / (ms * 1e-3));
  }
#define QD(ILP) for (int bpsm : {1, 2, 4}) { int blocks = sms * bpsm, thr = 128; \
    float ms = timeit([&] { tput_qd<ILP><<<blocks, thr>>>(d, IT / 4, 2.0, 0.5, 0.3); }); \
    double ops = (double)blocks * thr * (IT / 4) * ILP; printf(",\"qd_steps_per_s_ilp%d_w%d\":%.4e", ILP, bpsm * 4, ops / (ms * 1e-3)); }
#define PJ(ILP) for (int bpsm : {1, 2, 4}) { int blocks = sms * bpsm, thr = 128; \
    float ms = timeit([&] { tput_proj<ILP><<<blocks, thr>>>(d, IT / 4, 2.0, 0.5, 0.3); }); \
    double ops = (double)blocks * thr * (IT / 4) * ILP; printf(",\"proj_steps_per_s_ilp%d_w%d\":%.4e", ILP, bpsm * 4, ops / (ms * 1e-3)); }
  QD(1) QD(2) QD(4) PJ(1) PJ(2) PJ(4) PJ(8)
  printf("}\n");
  return 0;
}
