// Microbenchmark: interval multiply-add throughput of the band forms (kernels.cuh).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_10868_b200/csrc/kernels.cuh"
#include "../../paper_2007_10868_b200/csrc/numeric.cuh"
using namespace pc;

template <int ILP, int V>
__global__ void thr(double* out, const double* t, const double* w, int n) {
  double lo[ILP], hi[ILP];
  bool bad = false;
  for (int u = 0; u < ILP; ++u) lo[u] = hi[u] = 0.0;
  for (int i = 0; i < n; ++i) {
    const double ww = w[i & 255];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const double c = t[(i + u) & 255], c2 = t[(i + u + 7) & 255];
      if (V == 0) madd_band(ww, c, c2, lo[u], hi[u]);
      else if (V == 1) madd_band_lat(ww, c, c2, lo[u], hi[u]);
      else { lo[u] = f_add_dn(lo[u], f_mul_dn(c, ww, bad)); hi[u] = f_add_up(hi[u], f_mul_up(c2, ww, bad)); }
    }
  }
  double s = bad;
  for (int u = 0; u < ILP; ++u) s += lo[u] + hi[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP, int V>
void run(const char* name, double* out, double* t, double* w, int nsm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 2048;
  for (int bps : {2, 4, 8}) {
    dim3 g(nsm * bps);
    thr<ILP, V><<<g, 256>>>(out, t, w, n); cudaDeviceSynchronize();
    cudaEventRecord(e0); thr<ILP, V><<<g, 256>>>(out, t, w, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-10s ILP%d %d blk/SM: %.3e madds/s\n", name, ILP, bps, (double)g.x * 256 * ILP * n / (ms * 1e-3));
  }
}

int main() {
  double *t, *w, *out;
  cudaMalloc(&t, 2048); cudaMalloc(&w, 2048); cudaMalloc(&out, 1 << 24);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1e-3 * (i + 1) / 3.0 * ((i & 1) ? -1 : 1);
  cudaMemcpy(t, h, 2048, cudaMemcpyHostToDevice); cudaMemcpy(w, h, 2048, cudaMemcpyHostToDevice);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<1, 0>("band", out, t, w, nsm); run<4, 0>("band", out, t, w, nsm);
  run<1, 1>("band_lat", out, t, w, nsm); run<4, 1>("band_lat", out, t, w, nsm);
  run<4, 2>("checked", out, t, w, nsm);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
