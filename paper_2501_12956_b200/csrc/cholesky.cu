// cholesky.cu -- preconditioning (App. A Eqs. 23-24; Remark 1),
// the fp64 Cholesky factor H' = L L^T (Eq. 9; Algorithm 1), and the
// fp32 operands the S- and T-updates read (reading R-10).
//
// Factorisation: right-looking blocked Cholesky with NB = 64, in place on the lower
// triangle of A (fp64).  Per block column k: (1) one CTA factors the 64 x 64 diagonal
// block in shared memory, (2) TRSM of the panel below it (one warp per row, forward
// substitution, the 64 x 64 factor in shared memory), (3) trailing SYRK update of the
// lower tiles (64 x 64 tiles, 4 x 4 fp64 register blocking, K = 64).  Each tile has one
// owner per step, so the result is deterministic (bitwise identical on every rank).
// A non-positive pivot records its global index (atomicMin) in *d_status.
#include <float.h>
#include <limits.h>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int NB = 64;
constexpr int LDS = NB + 1;  // padded fp64 row stride in shared memory

// ---------------------------------------------------------------- precondition
// delta_i = max(sum_j |H_ij| - 2 H_ii, 1e-8) + tau * mean(diag H)   (ADAPTIVE, Eq. 23 + R-3)
// delta_i = lambda                                                  (FIXED_LAMBDA)
// delta_i = 0                                                        (NONE)
__global__ void diag_mean_kernel(const double* __restrict__ H, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += H[i * n + i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s / (double)n;
  }
}

// One warp per row: A = H (full row copy) with A_ii += delta_i.
__global__ void precondition_kernel(const double* __restrict__ H, int64_t n, int policy,
                                    double lambda, double tau, const double* __restrict__ diag_mean,
                                    double* __restrict__ A, double* __restrict__ delta) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double* h = H + i * n;
  double* a = A + i * n;
  double rs = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    const double v = h[j];
    a[j] = v;
    rs += fabs(v);
  }
  for (int o = 16; o; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  if (lane == 0) {
    double d = 0.0;
    if (policy == GANQ_PRECOND_ADAPTIVE) {
      d = rs - 2.0 * h[i];
      if (d < 1e-8) d = 1e-8;
      d += tau * (*diag_mean);
    } else if (policy == GANQ_PRECOND_FIXED_LAMBDA) {
      d = lambda;
    }
    a[i] = h[i] + d;
    if (delta) delta[i] = d;
  }
}

// ---------------------------------------------------------------- diagonal block
// One CTA of 256 threads = 16 x 16; thread (tx, ty) owns the 4 x 4 elements
// (ty + 16 a, tx + 16 b) of the 64 x 64 block (no integer division in the loops).
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ A, int64_t n, int64_t k0,
                                                         int* __restrict__ status) {
  __shared__ double s[NB * LDS];
  const int kb = (int)min((int64_t)NB, n - k0);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, c = tx + 16 * b;
      s[r * LDS + c] = (r < kb && c <= r) ? A[(k0 + r) * n + k0 + c] : (r == c ? 1.0 : 0.0);
    }
  __syncthreads();
  for (int c = 0; c < kb; ++c) {
    double piv = s[c * LDS + c];
    if (!(piv > 0.0)) {  // not positive definite (or NaN)
      if (threadIdx.x == 0) atomicMin(status, (int)(k0 + c));
      piv = 1.0;
    }
    const double inv = 1.0 / sqrt(piv);
    __syncthreads();  // everyone has read the pivot
    // scale column c below the diagonal; the diagonal becomes sqrt(piv)
    if (threadIdx.x < NB) {
      const int r = threadIdx.x;
      if (r > c) s[r * LDS + c] *= inv;
      if (r == c) s[r * LDS + c] = piv * inv;
    }
    __syncthreads();
    // trailing rank-1 update of the lower part (rows, cols > c)
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = ty + 16 * a;
      if (r <= c) continue;
      const double lrc = s[r * LDS + c];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = tx + 16 * b;
        if (q > c && q <= r) s[r * LDS + q] -= lrc * s[q * LDS + c];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, c = tx + 16 * b;
      if (r < kb && c <= r) A[(k0 + r) * n + k0 + c] = s[r * LDS + c];
    }
}

// ---------------------------------------------------------------- panel TRSM
// For rows r >= k0 + kb:  L[r, k0:k0+kb] = A[r, k0:k0+kb] * L_kk^{-T}  (forward substitution).
__global__ void __launch_bounds__(256) trsm_panel_kernel(double* __restrict__ A, int64_t n, int64_t k0) {
  __shared__ double s[NB * LDS];
  const int kb = (int)min((int64_t)NB, n - k0);
  for (int r = threadIdx.x >> 6; r < kb; r += 4) {
    const int c = threadIdx.x & 63;
    if (c < kb) s[r * LDS + c] = (c <= r) ? A[(k0 + r) * n + k0 + c] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t row = k0 + kb + (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  double* a = A + row * n + k0;
  double x0 = (lane < kb) ? a[lane] : 0.0;
  double x1 = (lane + 32 < kb) ? a[lane + 32] : 0.0;
  for (int c = 0; c < kb; ++c) {
    const double own = (c < 32) ? x0 : x1;
    double xc = __shfl_sync(0xffffffffu, own, c & 31);
    xc /= s[c * LDS + c];
    if (lane == (c & 31)) { if (c < 32) x0 = xc; else x1 = xc; }
    if (lane > c) x0 -= xc * s[lane * LDS + c];
    if (lane + 32 > c && lane + 32 < kb) x1 -= xc * s[(lane + 32) * LDS + c];
  }
  if (lane < kb) a[lane] = x0;
  if (lane + 32 < kb) a[lane + 32] = x1;
}

// ---------------------------------------------------------------- trailing SYRK
// A[i, j] -= sum_c L[i, k0+c] L[j, k0+c] for the lower tiles of the trailing matrix.
__global__ void __launch_bounds__(256) syrk_trailing_kernel(double* __restrict__ A, int64_t n,
                                                            int64_t k0) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (tj > ti) return;
  extern __shared__ double syrk_smem[];
  double* Pi = syrk_smem;
  double* Pj = syrk_smem + NB * LDS;
  const int64_t base = k0 + NB;  // first trailing row/col (only called when k0 + NB < n)
  const int64_t i0 = base + (int64_t)ti * NB, j0 = base + (int64_t)tj * NB;
  for (int r = threadIdx.x >> 6; r < NB; r += 4) {
    const int c = threadIdx.x & 63;
    Pi[r * LDS + c] = (i0 + r < n) ? A[(i0 + r) * n + k0 + c] : 0.0;
    Pj[r * LDS + c] = (j0 + r < n) ? A[(j0 + r) * n + k0 + c] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
#pragma unroll 4
  for (int c = 0; c < NB; ++c) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = Pi[(ty + 16 * q) * LDS + c];
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = Pj[(tx + 16 * q) * LDS + c];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t i = i0 + ty + 16 * x, j = j0 + tx + 16 * y;
      if (i < n && j <= i) A[i * n + j] -= acc[x][y];
    }
}

__global__ void zero_upper_kernel(double* __restrict__ A, int64_t n) {
  const int64_t total = n * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx % n;
    if (j > i) A[idx] = 0.0;
  }
}

// ---------------------------------------------------------------- derived fp32 operands
// Lhat[u][j] = L_uj / L_jj for u > j, 0 otherwise (the S-update's scaled feedback
// weights, reading R-10); H32 = fp32(H) for the T-update (reading R-4: raw H).
__global__ void derive_kernel(const double* __restrict__ L, const double* __restrict__ H, int64_t n,
                              float* __restrict__ Lhat, float* __restrict__ H32) {
  const int64_t total = n * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = idx / n, j = idx % n;
    if (Lhat) Lhat[idx] = (u > j) ? (float)(L[idx] / L[j * n + j]) : 0.0f;
    if (H32) H32[idx] = (float)H[idx];
  }
}

}  // namespace

ganq_status_t launch_precondition(const double* H, int64_t n, int policy, double lambda, double tau,
                                  double* A, double* delta, double* d_mean, cudaStream_t st) {
  diag_mean_kernel<<<1, 1024, 0, st>>>(H, n, d_mean);
  GANQ_LAUNCH_CHECK("diag_mean_kernel");
  precondition_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(H, n, policy, lambda, tau, d_mean, A,
                                                               delta);
  GANQ_LAUNCH_CHECK("precondition_kernel");
  return GANQ_OK;
}

ganq_status_t launch_cholesky(double* A, int64_t n, int* d_status, cudaStream_t st) {
  constexpr int kSyrkSmem = 2 * NB * LDS * sizeof(double);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(syrk_trailing_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSyrkSmem));
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    potrf_diag_kernel<<<1, 256, 0, st>>>(A, n, k0, d_status);
    GANQ_LAUNCH_CHECK("potrf_diag_kernel");
    const int64_t rest = n - k0 - NB;
    if (rest <= 0) break;
    trsm_panel_kernel<<<(unsigned)((rest + 7) / 8), 256, 0, st>>>(A, n, k0);
    GANQ_LAUNCH_CHECK("trsm_panel_kernel");
    const unsigned T = (unsigned)((rest + NB - 1) / NB);
    syrk_trailing_kernel<<<dim3(T, T), 256, kSyrkSmem, st>>>(A, n, k0);
    GANQ_LAUNCH_CHECK("syrk_trailing_kernel");
  }
  zero_upper_kernel<<<1184, 256, 0, st>>>(A, n);
  GANQ_LAUNCH_CHECK("zero_upper_kernel");
  return GANQ_OK;
}

ganq_status_t launch_derive_operands(const double* L, const double* H, int64_t n, float* Lhat,
                                     float* H32, cudaStream_t st) {
  derive_kernel<<<1184, 256, 0, st>>>(L, H, n, Lhat, H32);
  GANQ_LAUNCH_CHECK("derive_kernel");
  return GANQ_OK;
}

}  // namespace ganq
