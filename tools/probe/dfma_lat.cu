// Microbenchmark: latency of a dependent fp64 FMA chain and of MUFU.RCP64H+Newton division on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_div(double* out, long long* cyc, double a, int n) {
  double x = out[threadIdx.x] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) x = a / x + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_mul(double* out, long long* cyc, double a, int n) {
  double x = out[threadIdx.x] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) x = x * a;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i + 1) % 1024;
  __syncwarp();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) idx = (int)s[idx];
  }
  long long t1 = clock64();
  out[threadIdx.x] = idx;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMemset(out, 0, 1024 * 8);
  cudaMalloc(&cyc, 8);
  long long h;
  const int n = 1000;
  lat<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
  lat<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent chain: %.2f clk per op\n", (double)h / (16.0 * n));
  lat_mul<<<1, 32>>>(out, cyc, 0.9999, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent chain: %.2f clk per op\n", (double)h / (16.0 * n));
  lat_div<<<1, 32>>>(out, cyc, 0.7, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("fp64 a/x+1 dependent chain: %.2f clk per op\n", (double)h / (16.0 * n));
  lat_lds<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 + F2I dependent chain: %.2f clk per op\n", (double)h / (16.0 * n));
  return 0;
}
