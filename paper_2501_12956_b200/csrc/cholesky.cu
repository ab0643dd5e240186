// cholesky.cu -- preconditioning (App. A Eqs. 23-24; Remark 1),
// the fp64 Cholesky factor H' = L L^T (Eq. 9; Algorithm 1), and the
// fp32 operands the S- and T-updates read (reading R-10).
//
// Factorisation: right-looking blocked Cholesky with NB = 64, in place on the lower
// triangle of A (fp64).  Per block column k: (1) one CTA factors the 64 x 64 diagonal
// block in shared memory, (2) TRSM of the panel below it (thread per row, forward
// substitution from shared memory), (3) trailing SYRK update of the lower tiles (128 x 128
// tiles, 8 x 8 fp64 register blocking), applied once per two panels (K = 128).  Each tile has
// one owner per step, so the result is deterministic (bitwise identical on every rank).
// A non-positive pivot records its global index (atomicMin) in *d_status.
#include <float.h>
#include <limits.h>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int NB = 64;
constexpr int LDS = NB + 1;  // padded fp64 row stride in shared memory

// 8-byte global -> shared copy that does not hold a register (all of a tile's copies are in
// flight together; cp_wait() before the barrier that publishes them)
__device__ __forceinline__ void cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

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
// (ty + 16 a, tx + 16 b) of the 64 x 64 block.  Unscaled elimination with one barrier per
// column: step c subtracts a_rc a_qc / d_c from the trailing elements (d_c = a_cc, the pivot),
// which equals L_rc L_qc of the standard algorithm; afterwards L_rc = a_rc / sqrt(d_c).
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ A, int64_t n, int64_t k0,
                                                         int* __restrict__ status) {
  extern __shared__ double potrf_smem[];
  double* s = potrf_smem;               // [64][LDS] the block
  double* dpiv = potrf_smem + NB * LDS; // [64] pivots
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
  for (int c = 0; c < NB; ++c) {
    double d = s[c * LDS + c];
    if (!(d > 0.0)) {  // not positive definite (or NaN)
      if (threadIdx.x == 0 && c < kb) atomicMin(status, (int)(k0 + c));
      d = 1.0;
    }
    if (threadIdx.x == 0) dpiv[c] = d;
    const double id = 1.0 / d;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = ty + 16 * a;
      if (r <= c) continue;
      const double arc = s[r * LDS + c] * id;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = tx + 16 * b;
        if (q > c && q <= r) s[r * LDS + q] -= arc * s[q * LDS + c];
      }
    }
    __syncthreads();
  }
  // L_rc = a_rc / sqrt(d_c), L_cc = sqrt(d_c)
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, c = tx + 16 * b;
      const double sd = sqrt(dpiv[c]);
      if (c < r) s[r * LDS + c] /= sd;
      else if (c == r) s[r * LDS + c] = sd;
    }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, c = tx + 16 * b;
      if (r < kb && c <= r) A[(k0 + r) * n + k0 + c] = s[r * LDS + c];
    }
}

// ---------------------------------------------------------------- panel TRSM
// For rows i >= k0 + kb:  x = L[i, k0:k0+kb] solves x L_kk^T = A[i, k0:k0+kb], i.e. forward
// substitution x_c = (a_c - sum_{q<c} x_q L_cq) / L_cc.  One thread per row (x in registers,
// four interleaved partial sums per column), 128 rows per CTA staged through shared memory
// (coalesced cp.async), L_kk in shared memory (broadcast reads).
constexpr int TR = 128;
__global__ void __launch_bounds__(TR) trsm_panel_kernel(double* __restrict__ A, int64_t n, int64_t k0) {
  extern __shared__ double trsm_smem[];
  double* Pr = trsm_smem;             // [TR][LDS] the CTA's panel rows
  double* Lk = trsm_smem + TR * LDS;  // [NB][LDS] L_kk
  double* rd = Lk + NB * LDS;         // [NB] 1 / L_cc
  const int kb = (int)min((int64_t)NB, n - k0);
  const int64_t i0 = k0 + kb + (int64_t)blockIdx.x * TR;
  for (int e = threadIdx.x; e < TR * NB; e += TR) {
    const int r = e >> 6, c = e & 63;
    if (i0 + r < n && c < kb) cp8(&Pr[r * LDS + c], &A[(i0 + r) * n + k0 + c]);
    else Pr[r * LDS + c] = 0.0;
  }
  for (int e = threadIdx.x; e < NB * NB; e += TR) {
    const int r = e >> 6, c = e & 63;
    if (r < kb && c <= r) cp8(&Lk[r * LDS + c], &A[(k0 + r) * n + k0 + c]);
    else Lk[r * LDS + c] = (r == c) ? 1.0 : 0.0;
  }
  cp_wait();
  __syncthreads();
  if (threadIdx.x < NB) rd[threadIdx.x] = 1.0 / Lk[threadIdx.x * LDS + threadIdx.x];
  __syncthreads();
  const int r = threadIdx.x;
  double x[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    double p0 = Pr[r * LDS + c], p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
    for (int q = 0; q + 3 < c; q += 4) {
      p0 = fma(-x[q], Lk[c * LDS + q], p0);
      p1 = fma(-x[q + 1], Lk[c * LDS + q + 1], p1);
      p2 = fma(-x[q + 2], Lk[c * LDS + q + 2], p2);
      p3 = fma(-x[q + 3], Lk[c * LDS + q + 3], p3);
    }
#pragma unroll
    for (int q = c & ~3; q < c; ++q) p0 = fma(-x[q], Lk[c * LDS + q], p0);
    x[c] = ((p0 + p1) + (p2 + p3)) * rd[c];
  }
  const int64_t i = i0 + r;
  if (i < n) {
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c < kb) A[i * n + k0 + c] = x[c];
  }
}

// ---------------------------------------------------------------- trailing SYRK
// A[i, j] -= sum_c L[i, k0+c] L[j, k0+c] for the lower 128 x 128 tiles of the trailing matrix;
// thread (tx, ty) owns the 8 x 8 elements (ty + 16 x, tx + 16 y) of its tile.
constexpr int ST = 128;  // SYRK tile
// A[i, j] -= sum_{c in [k0, k0 + kw)} L[i, c] L[j, c] for base <= j <= i < n, j < cend: the lower
// 128 x 128 tiles of the trailing block, the kw <= 128 panel columns streamed through shared
// memory in chunks of 64 (the accumulators stay in registers, one read-modify-write per tile).
__global__ void __launch_bounds__(256) syrk_trailing_kernel(double* __restrict__ A, int64_t n, int64_t k0,
                                                            int kw, int64_t base, int64_t cend) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (tj > ti) return;
  extern __shared__ double syrk_smem[];
  double* Pi = syrk_smem;
  double* Pj = syrk_smem + ST * LDS;
  const int64_t i0 = base + (int64_t)ti * ST, j0 = base + (int64_t)tj * ST;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[8][8] = {};
  for (int kc = 0; kc < kw; kc += NB) {
    const int kcw = min(NB, kw - kc);
    if (kc > 0) __syncthreads();  // the previous chunk has been consumed
    for (int e = threadIdx.x; e < ST * NB; e += 256) {
      const int r = e >> 6, c = e & 63;
      if (i0 + r < n && c < kcw) cp8(&Pi[r * LDS + c], &A[(i0 + r) * n + k0 + kc + c]);
      else Pi[r * LDS + c] = 0.0;
      if (j0 + r < cend && c < kcw) cp8(&Pj[r * LDS + c], &A[(j0 + r) * n + k0 + kc + c]);
      else Pj[r * LDS + c] = 0.0;
    }
    cp_wait();
    __syncthreads();
#pragma unroll 2
    for (int c = 0; c < NB; ++c) {
      double a[8], b[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = Pi[(ty + 16 * q) * LDS + c];
#pragma unroll
      for (int q = 0; q < 8; ++q) b[q] = Pj[(tx + 16 * q) * LDS + c];
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
  }
  // read-modify-write in two batches of 32: all loads of a batch are issued before its stores
  // (the compiler keeps loads and stores through one pointer in order, one round trip each)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double old[4][8];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const int64_t i = i0 + ty + 16 * (4 * h + x), j = j0 + tx + 16 * y;
        old[x][y] = (i < n && j <= i && j < cend) ? A[i * n + j] : 0.0;
      }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const int64_t i = i0 + ty + 16 * (4 * h + x), j = j0 + tx + 16 * y;
        if (i < n && j <= i && j < cend) A[i * n + j] = old[x][y] - acc[4 * h + x][y];
      }
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

// Side stream and events of the Cholesky look-ahead, created once per host thread and device.
struct LookAhead {
  int device = -1;
  cudaStream_t side = nullptr;
  cudaEvent_t th = nullptr, tr = nullptr;
};
LookAhead& look_ahead() {
  static thread_local LookAhead la;
  int dev = 0;
  cudaGetDevice(&dev);
  if (la.device != dev) {
    // highest priority: the side stream's panel kernels take SMs as soon as bulk-update CTAs
    // retire instead of queueing behind the bulk kernel's remaining CTAs
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&la.side, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&la.th, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&la.tr, cudaEventDisableTiming);
    la.device = dev;
  }
  return la;
}

ganq_status_t launch_cholesky(double* A, int64_t n, int* d_status, cudaStream_t st) {
  constexpr int kSyrkSmem = 2 * ST * LDS * sizeof(double);
  constexpr int kTrsmSmem = ((TR + NB) * LDS + NB) * sizeof(double);
  constexpr int kPotrfSmem = (NB * LDS + NB) * sizeof(double);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotrfSmem));
  GANQ_CUDA_TRY(cudaFuncSetAttribute(syrk_trailing_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSyrkSmem));
  GANQ_CUDA_TRY(cudaFuncSetAttribute(trsm_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmSmem));
  auto panel = [&](int64_t k0, cudaStream_t ps) -> ganq_status_t {
    potrf_diag_kernel<<<1, 256, kPotrfSmem, ps>>>(A, n, k0, d_status);
    GANQ_LAUNCH_CHECK("potrf_diag_kernel");
    const int64_t rest = n - k0 - NB;
    if (rest > 0) {
      trsm_panel_kernel<<<(unsigned)((rest + TR - 1) / TR), TR, kTrsmSmem, ps>>>(A, n, k0);
      GANQ_LAUNCH_CHECK("trsm_panel_kernel");
    }
    return GANQ_OK;
  };
  auto syrk = [&](int64_t k0, int kw, int64_t base, int64_t cend) -> ganq_status_t {
    const unsigned Ti = (unsigned)((n - base + ST - 1) / ST), Tj = (unsigned)((cend - base + ST - 1) / ST);
    syrk_trailing_kernel<<<dim3(Tj, Ti), 256, kSyrkSmem, st>>>(A, n, k0, kw, base, cend);
    GANQ_LAUNCH_CHECK("syrk_trailing_kernel");
    return GANQ_OK;
  };
  if (n < 6144) {
    // One panel per pass with look-ahead: the trailing update of panel k is split into a thin
    // update of panel k+1's columns and the bulk (columns beyond); panel k+1's diagonal factor
    // and TRSM run on a side stream while the bulk update of panel k runs on `st`.
    //   side:  potrf(k+1), trsm(k+1)    after thin(k)          (event th)
    //   st:    thin(k+1)                after trsm(k+1)        (event tr)
    // thin(k) follows bulk(k-1) on st, so panel k+1 has every earlier update when it starts.
    LookAhead& la = look_ahead();
    GANQ_CUDA_TRY(cudaEventRecord(la.th, st));
    GANQ_CUDA_TRY(cudaStreamWaitEvent(la.side, la.th, 0));
    ganq_status_t s;
    if ((s = panel(0, la.side))) return s;
    GANQ_CUDA_TRY(cudaEventRecord(la.tr, la.side));
    for (int64_t k0 = 0; k0 < n; k0 += NB) {
      const int64_t k1 = k0 + NB;
      if (k1 >= n) break;
      GANQ_CUDA_TRY(cudaStreamWaitEvent(st, la.tr, 0));  // trsm(k) done
      if ((s = syrk(k0, NB, k1, min(k1 + NB, n)))) return s;  // thin(k): panel k+1's columns
      GANQ_CUDA_TRY(cudaEventRecord(la.th, st));
      GANQ_CUDA_TRY(cudaStreamWaitEvent(la.side, la.th, 0));
      if ((s = panel(k1, la.side))) return s;                // overlaps bulk(k) below
      GANQ_CUDA_TRY(cudaEventRecord(la.tr, la.side));
      if (k1 + NB < n)
        if ((s = syrk(k0, NB, k1 + NB, n))) return s;        // bulk(k)
    }
    GANQ_CUDA_TRY(cudaStreamWaitEvent(st, la.tr, 0));      // the last panel is factored
  } else {
    // large n: two panels per pass -- factor panel k, update only panel k + 1's columns (thin
    // SYRK), factor panel k + 1, then one trailing SYRK with both panels (K = 128): the trailing
    // matrix (beyond L2) is read and written once per 128 columns.  (Look-ahead on the side
    // stream was measured slower here: the HBM-bound bulk update loses SMs to the panel kernels.)
    for (int64_t k0 = 0; k0 < n; k0 += 2 * NB) {
      ganq_status_t s;
      if ((s = panel(k0, st))) return s;
      const int64_t k1 = k0 + NB;
      if (k1 >= n) break;
      if ((s = syrk(k0, NB, k1, min(k1 + NB, n)))) return s;  // panel k+1's columns only
      if ((s = panel(k1, st))) return s;
      const int64_t base = k1 + NB;
      if (base >= n) break;
      if ((s = syrk(k0, 2 * NB, base, n))) return s;          // trailing block, both panels
    }
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
