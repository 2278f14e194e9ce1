// Microbenchmark: dependent-chain latency and throughput of the emulated
// directed-rounding ops (numeric.cuh) on sm_100a. Not product code.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_10868_b200/csrc/numeric.cuh"
using namespace pc;

#define N_STEPS 4096

__global__ void lat_dadd(double* out, const double* t, int n) {
  double acc = t[threadIdx.x];
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, t[i & 255]);
  out[threadIdx.x] = acc;
}
__global__ void lat_fadd_dn(double* out, const double* t, int n) {
  double acc = t[threadIdx.x];
  for (int i = 0; i < n; ++i) acc = f_add_dn(acc, t[i & 255]);
  out[threadIdx.x] = acc;
}
// candidate: integer nextdown step
__device__ __forceinline__ double g_add_dn(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double rd = __dadd_rd(a, b), ru = __dadd_ru(a, b);
  long long bs = __double_as_longlong(s);
  const long long st = bs + ((bs < 0) ? 1 : -1);  // s never 0 when inexact
  return (rd == ru) ? s : __longlong_as_double(st);
}
__global__ void lat_gadd_dn(double* out, const double* t, int n) {
  double acc = t[threadIdx.x];
  for (int i = 0; i < n; ++i) acc = g_add_dn(acc, t[i & 255]);
  out[threadIdx.x] = acc;
}
// candidate: result from rd/ru only: inexact & s==rd -> nextdown(rd) else rd
__device__ __forceinline__ double h_add_dn(double a, double b) {
  const double rd = __dadd_rd(a, b), ru = __dadd_ru(a, b), s = __dadd_rn(a, b);
  const long long b2 = __double_as_longlong(rd);
  const double nd = __longlong_as_double(b2 + ((b2 < 0) ? 1 : -1));
  return (rd != ru && s == rd) ? nd : rd;
}
__global__ void lat_hadd_dn(double* out, const double* t, int n) {
  double acc = t[threadIdx.x];
  for (int i = 0; i < n; ++i) acc = h_add_dn(acc, t[i & 255]);
  out[threadIdx.x] = acc;
}
// throughput: many independent chains per thread, all warps
template <int ILP>
__global__ void thr_madd(double* out, const double* t, const double* w, int n) {
  double lo[ILP], hi[ILP];
  bool bad = false;
  for (int u = 0; u < ILP; ++u) lo[u] = hi[u] = t[(threadIdx.x + u) & 255];
  for (int i = 0; i < n; ++i) {
    const double ww = w[i & 255];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const double c = t[(i + u) & 255];
      lo[u] = f_add_dn(lo[u], f_mul_dn(c, ww, bad));
      hi[u] = f_add_up(hi[u], f_mul_up(c, ww, bad));
    }
  }
  double s = bad;
  for (int u = 0; u < ILP; ++u) s += lo[u] + hi[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void thr_dfma(double* out, const double* t, int n) {
  double a[8];
  for (int u = 0; u < 8; ++u) a[u] = t[(threadIdx.x + u) & 255];
  const double x = t[3], y = t[5];
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __fma_rn(a[u], x, y);
  double s = 0;
  for (int u = 0; u < 8; ++u) s += a[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *t, *w, *out;
  cudaMalloc(&t, 256 * 8); cudaMalloc(&w, 256 * 8); cudaMalloc(&out, 1 << 24);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1e-3 * (i + 1) / 3.0 * ((i & 1) ? -1 : 1);
  cudaMemcpy(t, h, 2048, cudaMemcpyHostToDevice);
  cudaMemcpy(w, h, 2048, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  auto lat = [&](const char* name, void (*k)(double*, const double*, int)) {
    k<<<1, 32>>>(out, t, N_STEPS); cudaDeviceSynchronize();
    cudaEventRecord(e0); k<<<1, 32>>>(out, t, N_STEPS); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-12s %.2f ns/step (%.1f cycles at %d MHz)\n", name, ms * 1e6 / N_STEPS, ms * 1e6 / N_STEPS * clk / 1e6, clk / 1000);
  };
  lat("dadd", lat_dadd); lat("f_add_dn", lat_fadd_dn); lat("g_add_dn", lat_gadd_dn); lat("h_add_dn", lat_hadd_dn);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    const int n = 2048;
    dim3 g(nsm * blocks_per_sm);
    thr_madd<4><<<g, 256>>>(out, t, w, n); cudaDeviceSynchronize();
    cudaEventRecord(e0); thr_madd<4><<<g, 256>>>(out, t, w, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double madds = (double)g.x * 256 * 4 * n;
    printf("madd ILP4 %d blk/SM x256: %.3e interval madds/s\n", blocks_per_sm, madds / (ms * 1e-3));
  }
  {
    const int n = 4096; dim3 g(nsm * 8);
    thr_dfma<<<g, 256>>>(out, t, n); cudaDeviceSynchronize();
    cudaEventRecord(e0); thr_dfma<<<g, 256>>>(out, t, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("dfma: %.3e FMA/s (%.1f TFLOPS)\n", (double)g.x * 256 * 8 * n / (ms * 1e-3), 2.0 * g.x * 256 * 8 * n / (ms * 1e-3) / 1e12);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
