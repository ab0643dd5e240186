// outlier.cu -- NEXT-2, GANQ*: outlier extraction and weight decomposition, Algorithm 2
// (Appendix B; §3.3), and the sparse product of the deployed layer.
//
// Per row: the cutoffs are the row's order statistics at Algorithm 2's indices upper =
// floor(n p), lower = ceil(n (1 - p)), p = 1 - 0.5 r (0-based, reading R-21), found by an exact
// radix select on order-preserving uint32 keys (4 passes of 8 bits, both ranks together).  An
// entry is an outlier iff w >= c_upper or w <= c_lower (ties included, R-22); W_dense = W - W o M.
// The CSR of W o M lists each row's outliers in ascending column order.
#include <cuda_fp16.h>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

constexpr int OT = 256;  // threads per row-CTA

// rank k (0-based) of the keys in s[0, n) whose bits above `shift + 8` equal `prefix`: returns the
// 8-bit digit of the k-th smallest and updates k to its rank within that digit's bucket.
__device__ void select_digit(const int* hist, int& k, uint32_t& digit) {
  // one warp: lane l owns bins [8 l, 8 l + 8)
  const int lane = threadIdx.x & 31;
  int loc[8], sum = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) { loc[b] = hist[8 * lane + b]; sum += loc[b]; }
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  const int excl = inc - sum;
  const unsigned hit = __ballot_sync(0xffffffffu, excl <= k && k < inc);
  const int src = __ffs(hit) - 1;
  int d = 0, kk = k;
  if (lane == src) {
    kk = k - excl;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      if (kk < loc[b]) { d = 8 * lane + b; break; }
      kk -= loc[b];
    }
  }
  digit = (uint32_t)__shfl_sync(0xffffffffu, d, src);
  k = __shfl_sync(0xffffffffu, kk, src);
}

__global__ void __launch_bounds__(OT) outlier_split_kernel(const float* __restrict__ W, int64_t n, int64_t up,
                                                           int64_t lo, float* __restrict__ Wd,
                                                           float* __restrict__ c_lo, float* __restrict__ c_hi,
                                                           int64_t* __restrict__ counts) {
  extern __shared__ uint32_t keys[];
  __shared__ int hist[2][256];
  __shared__ uint32_t pref[2];
  __shared__ int red[OT / 32];
  const int64_t i = blockIdx.x;
  const float* w = W + i * n;
  for (int64_t j = threadIdx.x; j < n; j += OT) keys[j] = fkey(w[j]);
  int kr[2] = {(int)up, (int)lo};
  uint32_t prefix[2] = {0u, 0u};
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 512; b += OT) (&hist[0][0])[b] = 0;
    __syncthreads();
    const uint32_t hmask = (shift == 24) ? 0u : (0xffffffffu << (shift + 8));
    for (int64_t j = threadIdx.x; j < n; j += OT) {
      const uint32_t k = keys[j];
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if ((k & hmask) == prefix[t]) atomicAdd(&hist[t][(k >> shift) & 255u], 1);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp < 2) {
      uint32_t d;
      select_digit(hist[warp], kr[warp], d);
      if ((threadIdx.x & 31) == 0) pref[warp] = prefix[warp] | (d << shift);
    }
    __syncthreads();
    prefix[0] = pref[0];
    prefix[1] = pref[1];
    // (kr of the other warps is stale but unused; warp t carries rank t)
  }
  const float chi = unkey(prefix[0]), clo = unkey(prefix[1]);
  if (threadIdx.x == 0) {
    c_hi[i] = chi;
    c_lo[i] = clo;
  }
  int cnt = 0;
  for (int64_t j = threadIdx.x; j < n; j += OT) {
    const float x = w[j];
    const bool o = (x >= chi) || (x <= clo);
    const float ws = o ? x : 0.0f;  // W o M
    Wd[i * n + j] = __fsub_rn(x, ws);
    cnt += o;
  }
  for (int o2 = 16; o2; o2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o2);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int q = 0; q < OT / 32; ++q) s += red[q];
    counts[i] = s;
  }
}

// in place: offsets[1..m] hold the counts; exclusive -> inclusive prefix sums, offsets[0] = 0
__global__ void __launch_bounds__(1024) offsets_scan_kernel(int64_t* __restrict__ off, int64_t m) {
  __shared__ int64_t part[1024];
  const int64_t per = (m + 1023) / 1024;
  const int64_t a = 1 + threadIdx.x * per, b = min(m + 1, a + per);
  int64_t s = 0;
  for (int64_t q = a; q < b; ++q) s += off[q];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int q = 0; q < 1024; ++q) { const int64_t v = part[q]; part[q] = run; run += v; }
    off[0] = 0;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t q = a; q < b; ++q) { run += off[q]; off[q] = run; }
}

// warp per row: outliers in ascending column order (ballot compaction)
__global__ void outlier_csr_kernel(const float* __restrict__ W, int64_t m, int64_t n, const float* __restrict__ c_lo,
                                   const float* __restrict__ c_hi, const int64_t* __restrict__ off,
                                   int32_t* __restrict__ col, float* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= m) return;
  const float chi = c_hi[i], clo = c_lo[i];
  int64_t base = off[i];
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    const int64_t j = j0 + lane;
    const float x = (j < n) ? W[i * n + j] : 0.0f;
    const bool o = j < n && ((x >= chi) || (x <= clo));
    const unsigned bal = __ballot_sync(0xffffffffu, o);
    if (o) {
      const int64_t pos = base + __popc(bal & ((1u << lane) - 1u));
      col[pos] = (int32_t)j;
      val[pos] = x;
    }
    base += __popc(bal);
  }
}

// warp per row: Y[t][i] += sum_k val[k] X[t][col[k]] (fp32, lane-strided then butterfly)
__global__ void sparse_gemm_add_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                                       const float* __restrict__ val, int64_t m, int64_t n,
                                       const __half* __restrict__ X, int64_t p, float* __restrict__ Y) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= m) return;
  const int64_t a = off[i], b = off[i + 1];
  for (int64_t t = 0; t < p; ++t) {
    float acc = 0.0f;
    for (int64_t k = a + lane; k < b; k += 32) acc = fmaf(val[k], __half2float(X[t * n + col[k]]), acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) Y[t * m + i] += acc;
  }
}

}  // namespace

void outlier_indices(int64_t n, double r, int64_t* up, int64_t* lo) {
  const double p = 1.0 - 0.5 * r;  // Algorithm 2, tail percentile
  *up = (int64_t)floor((double)n * p);
  *lo = (int64_t)ceil((double)n * (1.0 - p));
}

ganq_status_t launch_outlier_split(const float* W, int64_t m, int64_t n, double r, float* Wd, float* c_lo,
                                   float* c_hi, int64_t* off, cudaStream_t st) {
  int64_t up, lo;
  outlier_indices(n, r, &up, &lo);
  const size_t smem = (size_t)n * sizeof(uint32_t);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(outlier_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  outlier_split_kernel<<<(unsigned)m, OT, smem, st>>>(W, n, up, lo, Wd, c_lo, c_hi, off + 1);
  GANQ_LAUNCH_CHECK("outlier_split_kernel");
  offsets_scan_kernel<<<1, 1024, 0, st>>>(off, m);
  GANQ_LAUNCH_CHECK("offsets_scan_kernel");
  return GANQ_OK;
}

ganq_status_t launch_outlier_csr(const float* W, int64_t m, int64_t n, const float* c_lo, const float* c_hi,
                                 const int64_t* off, int32_t* col, float* val, cudaStream_t st) {
  outlier_csr_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(W, m, n, c_lo, c_hi, off, col, val);
  GANQ_LAUNCH_CHECK("outlier_csr_kernel");
  return GANQ_OK;
}

ganq_status_t launch_sparse_gemm_add(const int64_t* off, const int32_t* col, const float* val, int64_t m, int64_t n,
                                     const uint16_t* X, int64_t p, float* Y, cudaStream_t st) {
  sparse_gemm_add_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(off, col, val, m, n,
                                                                   reinterpret_cast<const __half*>(X), p, Y);
  GANQ_LAUNCH_CHECK("sparse_gemm_add_kernel");
  return GANQ_OK;
}

}  // namespace ganq
