// microbenchmark: sustained fp64 FMA throughput (independent chains, all SMs)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, threads = 256, blocks = sms * 8;
  k<<<blocks, threads>>>(d, 10); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * iters * (double)threads * blocks;
  printf("fp64 FMA: %.2f TFLOP/s (%d SMs, %.3f ms)\n", flops / (ms * 1e-3) / 1e12, sms, ms);
  return 0;
}
