// validate.cu -- optional input validation (non-finite inputs are undefined
// behaviour; a debug run validates them).  Enabled per call by the environment variable
// GANQ_VALIDATE=1: ganq_hessian and ganq_quantize_layer then scan their inputs, synchronise, and
// return GANQ_ERR_INVALID_ARG naming the first non-finite element.  Off by default (no cost).
#include <stdlib.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

__device__ unsigned long long g_first_bad;

__device__ __forceinline__ bool bad(float v) { return !isfinite(v); }
__device__ __forceinline__ bool bad(double v) { return !isfinite(v); }
__device__ __forceinline__ bool bad(uint16_t v) { return (v & 0x7f80u) == 0x7f80u; }  // bf16 Inf / NaN

template <typename T>
__global__ void nonfinite_kernel(const T* __restrict__ x, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    if (bad(x[i])) atomicMin(&g_first_bad, (unsigned long long)i);
}

std::mutex g_validate_mu;

template <typename T>
ganq_status_t check(const T* x, int64_t rows, int64_t cols, const char* what, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_validate_mu);
  const unsigned long long none = ~0ull;
  GANQ_CUDA_TRY(cudaMemcpyToSymbolAsync(g_first_bad, &none, sizeof(none), 0, cudaMemcpyHostToDevice, st));
  nonfinite_kernel<T><<<1184, 256, 0, st>>>(x, rows * cols);
  GANQ_LAUNCH_CHECK("nonfinite_kernel");
  unsigned long long first = none;
  GANQ_CUDA_TRY(cudaMemcpyFromSymbolAsync(&first, g_first_bad, sizeof(first), 0, cudaMemcpyDeviceToHost, st));
  GANQ_CUDA_TRY(cudaStreamSynchronize(st));
  if (first != none) {
    set_error(GANQ_ERR_INVALID_ARG, "GANQ_VALIDATE: non-finite %s at (%lld, %lld)", what,
              (long long)(first / (unsigned long long)cols), (long long)(first % (unsigned long long)cols));
    set_error_index((int64_t)first);
    return GANQ_ERR_INVALID_ARG;
  }
  return GANQ_OK;
}

}  // namespace

bool validate_enabled() {
  const char* v = getenv("GANQ_VALIDATE");
  return v && atoi(v) != 0;
}

ganq_status_t validate_finite_f32(const float* x, int64_t rows, int64_t cols, const char* what, cudaStream_t st) {
  return check(x, rows, cols, what, st);
}
ganq_status_t validate_finite_f64(const double* x, int64_t rows, int64_t cols, const char* what, cudaStream_t st) {
  return check(x, rows, cols, what, st);
}
ganq_status_t validate_finite_bf16(const uint16_t* x, int64_t rows, int64_t cols, const char* what,
                                   cudaStream_t st) {
  return check(x, rows, cols, what, st);
}

}  // namespace ganq
