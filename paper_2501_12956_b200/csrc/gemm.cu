// gemm.cu -- fp32 contractions around the solver:
//   WH = W * H      (the W_i H S_i^T factor of Eq. 6, computed once per layer; W fixed)
//   EH = E * H      (objective, Eq. 8)   with E = W - W~ (residual kernel)
//   f_i = sum_j E_ij (EH)_ij in fp64 (rowdot kernel), f = sum_i f_i in fixed order.
// v1: register-blocked SIMT fp32 GEMM (128 x 128 tile, 8 x 8 per thread).
#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int TM = 128, TN = 128, TK = 16;

__global__ void __launch_bounds__(256)
gemm_f32_kernel(const float* __restrict__ A, const float* __restrict__ Bm, float* __restrict__ C,
                int64_t M, int64_t N, int64_t K) {
  __shared__ __align__(16) float As[TK][TM + 4];
  __shared__ __align__(16) float Bs[TK][TN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * TM, n0 = (int64_t)blockIdx.x * TN;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  for (int64_t k0 = 0; k0 < K; k0 += TK) {
    // A tile: 128 rows x 16 k -> As[k][row]
    for (int idx = threadIdx.x; idx < TM * TK; idx += 256) {
      const int r = idx / TK, kk = idx % TK;
      const int64_t gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? A[gm * K + gk] : 0.0f;
    }
    for (int idx = threadIdx.x; idx < TK * TN; idx += 256) {
      const int kk = idx / TN, c = idx % TN;
      const int64_t gk = k0 + kk, gn = n0 + c;
      Bs[kk][c] = (gk < K && gn < N) ? Bm[gk * N + gn] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 4 + 64]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4 + 64]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gn < N) C[gm * N + gn] = acc[i][j];
    }
  }
}

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

ganq_status_t launch_gemm_f32(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                              cudaStream_t st) {
  dim3 grid((unsigned)((N + TN - 1) / TN), (unsigned)((M + TM - 1) / TM));
  gemm_f32_kernel<<<grid, 256, 0, st>>>(A, B, C, M, N, K);
  GANQ_LAUNCH_CHECK("gemm_f32_kernel");
  return GANQ_OK;
}

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
