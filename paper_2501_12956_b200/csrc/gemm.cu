// gemm.cu -- the objective's elementwise parts (Eq. 8): E = W - W~ (residual kernel),
//   f_i = sum_j E_ij (EH)_ij in fp64 (rowdot kernel), f = sum_i f_i in fixed order (sum kernel).
// The contraction E H itself runs on the tensor cores (gemm_tc.cu).
#include "ganq_internal.cuh"

namespace ganq {
namespace {

__global__ void residual_kernel(const float* __restrict__ W, const uint8_t* __restrict__ Q,
                                const float* __restrict__ T, int64_t m, int64_t n, int nlev,
                                float* __restrict__ E) {
  const int64_t total = m * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n;
    E[idx] = __fsub_rn(W[idx], T[i * nlev + Q[idx]]);
  }
}

// one warp per row: per_row[i] = sum_j E_ij * EH_ij (fp64)
__global__ void rowdot_kernel(const float* __restrict__ E, const float* __restrict__ EH, int64_t m,
                              int64_t n, double* __restrict__ per_row) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  double s = 0.0;
  for (int64_t j = lane; j < n; j += 32) s += (double)E[row * n + j] * (double)EH[row * n + j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) per_row[row] = s;
}

// single block, fixed order: out = sum_i per_row[i]
__global__ void sum_kernel(const double* __restrict__ x, int64_t m, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += x[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

ganq_status_t launch_residual(const float* W, const uint8_t* Q, const float* T, int64_t m, int64_t n,
                              int nlev, float* E, cudaStream_t st) {
  residual_kernel<<<1184, 256, 0, st>>>(W, Q, T, m, n, nlev, E);
  GANQ_LAUNCH_CHECK("residual_kernel");
  return GANQ_OK;
}

ganq_status_t launch_rowdot(const float* E, const float* EH, int64_t m, int64_t n, double* per_row,
                            cudaStream_t st) {
  rowdot_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(E, EH, m, n, per_row);
  GANQ_LAUNCH_CHECK("rowdot_kernel");
  return GANQ_OK;
}

ganq_status_t launch_sum(const double* x, int64_t m, double* out, cudaStream_t st) {
  sum_kernel<<<1, 1024, 0, st>>>(x, m, out);
  GANQ_LAUNCH_CHECK("sum_kernel");
  return GANQ_OK;
}

}  // namespace ganq
