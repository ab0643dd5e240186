// Dependent-chain latencies on one warp (clock64): fp64 FMA, fp64 rcp estimate, fp32 FMA,
// shared-memory load, __syncthreads with 512 threads.   nvcc -arch=sm_100a -O3 lat.cu -o lat
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double x0, int iters) {
  __shared__ double sh[64];
  __shared__ int shi[64];
  if (threadIdx.x < 64) { sh[threadIdx.x] = x0; shi[threadIdx.x] = (threadIdx.x + 1) & 63; }
  __syncthreads();
  double x = x0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  double r = x;
  for (int i = 0; i < iters; ++i) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r)); r = y + 1e-300; }
  long long t2 = clock64();
  float f = (float)x0;
  for (int i = 0; i < iters; ++i) f = fmaf(f, 0.999999f, 1e-7f);
  long long t3 = clock64();
  int p = threadIdx.x & 63;
  for (int i = 0; i < iters; ++i) p = shi[p];
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t5 = clock64();
  double z = x0;
  for (int i = 0; i < iters; ++i) z = 1.0 / (z + 1.0);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
  out[threadIdx.x] = x + r + f + p + z + sh[p];
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
  const int iters = 4096;
  for (int threads : {32, 512}) {
    lat<<<1, threads>>>(out, cyc, 0.5, iters);
    lat<<<1, threads>>>(out, cyc, 0.5, iters);
    cudaDeviceSynchronize();
    printf("threads %d: dfma %.1f  drcp.approx %.1f  ffma %.1f  lds %.1f  syncthreads %.1f  ddiv %.1f cycles\n", threads,
           (double)cyc[0] / iters, (double)cyc[1] / iters, (double)cyc[2] / iters, (double)cyc[3] / iters,
           (double)cyc[4] / iters, (double)cyc[5] / iters);
  }
  return 0;
}
