// FP64 latency / throughput probe on the B200 (one-off microbenchmark, not product code):
// per-warp dependent DFMA chains with 1..32 independent chains per thread, 1..16 warps per
// SM (one CTA per SM), clock64 per warp. Prints clk per DFMA per chain and per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, long long* clk) {
  double a[CH];
  const double m = 1.0000001 + threadIdx.x * 1e-9, c = 1e-7;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = fma(a[i], m, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) clk[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}
__global__ void kcvt(double* out, int iters, long long* clk) {  // I2F.F64.S32 + DADD chain
  double a = threadIdx.x; int v = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) { a = (double)v + a; v = (int)__double2loint(a) & 1023; }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if ((threadIdx.x & 31) == 0) clk[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}
template <int CH>
void run(int warps, double* out, long long* clk) {
  const int iters = 2000;
  k<CH><<<148, warps * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  long long h[32 * 148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  printf("chains/thread %2d warps/SM %2d: %.2f clk per dependent DFMA, %.3f warp-DFMA/clk/SM\n", CH, warps,
         mx / iters, (double)warps * CH * iters / mx);
}
int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&clk, 148 * 32 * 8);
  for (int w : {1, 4, 8, 16}) { run<1>(w, out, clk); run<4>(w, out, clk); run<8>(w, out, clk); run<16>(w, out, clk); }
  kcvt<<<148, 32>>>(out, 2000, clk); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  printf("I2F.F64 + DADD + F2I-ish dependent chain: %.2f clk per iteration\n", h / 2000.0);
  return 0;
}
