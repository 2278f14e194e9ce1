// Microbenchmark: FP64 op throughput per rounding mode on sm_100a, and the
// band madd with register-resident operands (no loads in the loop).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_10868_b200/csrc/kernels.cuh"
using namespace pc;

template <int OP>
__global__ void ops(double* out, double seed, int n) {
  double x[8];
  for (int u = 0; u < 8; ++u) x[u] = seed * (threadIdx.x + u + 1);
  const double y = seed * 0.37, z = -seed * 1.7;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) x[u] = __dadd_rn(x[u], y);
      if (OP == 1) x[u] = __dadd_rd(x[u], y);
      if (OP == 2) x[u] = __dmul_rn(x[u], y);
      if (OP == 3) x[u] = __fma_rn(x[u], y, z);
      if (OP == 4) x[u] = __fma_rd(x[u], y, z);
      if (OP == 5) x[u] = __dmul_rd(x[u], y);
    }
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void madd(double* out, double seed, int n) {
  double lo[ILP], hi[ILP], c[ILP + 1];
  for (int u = 0; u < ILP; ++u) lo[u] = hi[u] = 0.0;
  for (int u = 0; u <= ILP; ++u) c[u] = seed * (threadIdx.x % 7 + u + 1) * (u & 1 ? -1 : 1);
  double w = seed * 0.3;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < ILP; ++u) madd_band(w, fmin(c[u], c[u + 1]), fmax(c[u], c[u + 1]), lo[u], hi[u]);
    w = __dmul_rn(w, -1.0000000001);
  }
  double s = 0;
  for (int u = 0; u < ILP; ++u) s += lo[u] + hi[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
double time_it(K k, int nsm, int bps, double* out, int n) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<nsm * bps, 256>>>(out, 1.0 / 3.0, n);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<<<nsm * bps, 256>>>(out, 1.0 / 3.0, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e-3;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 24);
  int nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 4096;
  const char* names[] = {"dadd.rn", "dadd.rd", "dmul.rn", "dfma.rn", "dfma.rd", "dmul.rd"};
  for (int bps : {4, 8}) {
    double t[6] = {time_it(ops<0>, nsm, bps, out, n), time_it(ops<1>, nsm, bps, out, n),
                   time_it(ops<2>, nsm, bps, out, n), time_it(ops<3>, nsm, bps, out, n),
                   time_it(ops<4>, nsm, bps, out, n), time_it(ops<5>, nsm, bps, out, n)};
    for (int o = 0; o < 6; ++o) {
      const double r = (double)nsm * bps * 256 * 8 * n / t[o];
      printf("%s %d blk/SM: %.3e ops/s = %.1f per SM per clk (at %d MHz)\n", names[o], bps, r,
             r / nsm / (clk * 1e3), clk / 1000);
    }
  }
  for (int bps : {2, 4, 8}) {
    const double t4 = time_it(madd<4>, nsm, bps, out, n), t8 = time_it(madd<8>, nsm, bps, out, n);
    printf("madd_band ILP4 %d blk/SM: %.3e madds/s; ILP8: %.3e madds/s\n", bps,
           (double)nsm * bps * 256 * 4 * n / t4, (double)nsm * bps * 256 * 8 * n / t8);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
