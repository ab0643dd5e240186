// Throughput of int32 -> fp32 conversions on sm_100a: I2F (the converter) vs the add-only
// 1.5 * 2^23 trick (integer add + fp32 add), per warp instruction, all warps of every SM busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cvt_rate cvt_rate.cu && ./cvt_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const int* __restrict__ in, float* out, int iters) {
  int x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = in[(threadIdx.x + u) & 255];
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float f;
      if (MODE == 0) f = (float)x[u];                                        // I2F
      else f = __int_as_float(x[u] + 0x4B400000) - 12582912.0f;             // VIADD + FADD
      acc += f;
      x[u] += 3;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int* in; float* out;
  cudaMalloc(&in, 1024); cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaMemset(in, 0, 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(in, out, iters); else k<1><<<blocks, threads>>>(in, out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double conv = (double)blocks * threads * iters * 8;
      if (rep) printf("%s: %.3f ms, %.1f conversions/clk/SM at 1.965 GHz\n", mode ? "add-only trick" : "I2F",
                      ms, conv / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
