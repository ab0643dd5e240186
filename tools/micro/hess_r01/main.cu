// Times the round-1 Hessian kernel (hessian_r01.cu, git 9cc7ad1) at c2 (n = 4096, p = 262144) in
// isolation, for comparison with the current one.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../../include main.cu hessian_r01.cu -lcuda -o hess_r01
#include <cstdio>
#include <cstdarg>
#include <cuda_runtime.h>
#include "../../../paper_2501_12956_b200/csrc/ganq_internal.cuh"
namespace ganq {
void set_error(ganq_status_t, const char* fmt, ...) { va_list ap; va_start(ap, fmt); vfprintf(stderr, fmt, ap); va_end(ap); }
void set_error_index(int64_t) {}
ganq_status_t cuda_fail(cudaError_t e, const char* w) { fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e)); return GANQ_ERR_CUDA; }
void count_launch() {}
ganq_status_t launch_hessian(const uint16_t* X, int64_t p, int64_t n, double* H, int accumulate, cudaStream_t st);
}
int main() {
  const int64_t n = 4096, p = 262144;
  uint16_t* X; double* H;
  cudaMalloc(&X, p * n * 2); cudaMalloc(&H, n * n * 8);
  cudaMemset(X, 0x3c, p * n * 2);  // bf16 ~ 0.0115 everywhere
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) ganq::launch_hessian(X, p, n, H, 0, 0);
  cudaDeviceSynchronize();
  // isolated launches separated by idle time (no power-cap build-up)
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); ganq::launch_hessian(X, p, n, H, 0, 0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("r01 hessian (syrk + mirror) best of 5: %.3f ms\n", best);
  return 0;
}
