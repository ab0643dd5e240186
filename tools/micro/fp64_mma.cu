// fp64 throughput at low occupancy: (1) 8x8 outer-product DFMA from registers (the SYRK inner
// loop without shared memory), (2) DMMA m8n8k4, (3) DMMA m16n8k4 -- 8 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void outer(double* out, int iters) {
  double acc[8][8] = {}, a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = 1e-9 * i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int y = 0; y < 8; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = a[i] * 1.0000001; }
  }
  double s = 0;
  for (int x = 0; x < 8; ++x) for (int y = 0; y < 8; ++y) s += acc[x][y];
  if (s == 12345.0) out[0] = s;
}
__global__ void dmma884(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void dmma1684(double* out, int iters) {
  double c[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = 2e-3, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.0) out[0] = s;
}
__global__ void dmma1688(double* out, int iters) {
  double c[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = 2e-3, a2 = 3e-3, a3 = 4e-3, b0 = 1e-9, b1 = 2e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.0) out[0] = s;
}
template <typename F>
void run(const char* name, F kern, double flops_per_thread_iter, int wps) {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000, threads = 32 * wps, blocks = sms;
  kern<<<blocks, threads>>>(d, 10); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = flops_per_thread_iter * iters * (double)threads * blocks;
  printf("%-10s %2d warps/SM: %.2f TFLOP/s (%.3f ms) err=%s\n", name, wps, flops / (ms * 1e-3) / 1e12, ms,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int w : {8, 16}) {
    run("outer8x8", outer, 2.0 * 64, w);
    run("dmma884", dmma884, 2.0 * 8 * 256 / 32, w);   // 8 MMAs x 8*8*4 FMAs per warp
    run("dmma1684", dmma1684, 2.0 * 8 * 512 / 32, w);
    run("dmma1688", dmma1688, 2.0 * 8 * 1024 / 32, w);
  }
  return 0;
}
