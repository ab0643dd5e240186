// kmeans.cu -- k-means initial codebook T^0 (NEXT-4, reading R-24): per-row 1-D Lloyd
// from the fp32 min-max grid (R-6).  One CTA per row; each iteration assigns every weight to its
// nearest level (fp64 distance of fp32 values -- exact; strict '<' scan keeps the first index on
// ties, R-7) and moves every non-empty level to the fp64 mean of its weights, rounded to fp32.
// Per-thread partial sums live in their own shared-memory column and are reduced in a fixed order,
// so the result is deterministic (and, the per-level sums being exact in fp64, bit-identical to a
// sequential sum).  The row (<= a few 10 KB) stays in L1 across the iterations.
#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int KM_THREADS = 128;
constexpr int KM_PARTS = 8;  // reduction: KM_PARTS groups of KM_THREADS / KM_PARTS threads

template <int NLEV>
__global__ void __launch_bounds__(KM_THREADS) kmeans_kernel(const float* __restrict__ W, int64_t n, int iters,
                                                            float* __restrict__ T) {
  __shared__ double acc[NLEV][KM_THREADS];
  __shared__ int cnt[NLEV][KM_THREADS];
  __shared__ double racc[NLEV][KM_PARTS];
  __shared__ int rcnt[NLEV][KM_PARTS];
  __shared__ double t[NLEV];
  const int tid = threadIdx.x;
  const int64_t row = blockIdx.x;
  const float* w = W + row * n;
  float* trow = T + row * NLEV;
  if (tid < NLEV) t[tid] = (double)trow[tid];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < NLEV; ++s) {
      acc[s][tid] = 0.0;
      cnt[s][tid] = 0;
    }
    __syncthreads();  // t[] of the previous iteration visible
    double tl[NLEV];
#pragma unroll
    for (int s = 0; s < NLEV; ++s) tl[s] = t[s];
    for (int64_t j = tid; j < n; j += KM_THREADS) {
      const double x = (double)__ldg(w + j);
      double best = fabs(x - tl[0]);
      int q = 0;
#pragma unroll
      for (int s = 1; s < NLEV; ++s) {
        const double d = fabs(x - tl[s]);
        const bool lt = d < best;
        best = lt ? d : best;
        q = lt ? s : q;
      }
      acc[q][tid] += x;
      cnt[q][tid] += 1;
    }
    __syncthreads();
    constexpr int SEG = KM_THREADS / KM_PARTS;
    for (int u = tid; u < NLEV * KM_PARTS; u += KM_THREADS) {
      const int s = u / KM_PARTS, part = u % KM_PARTS;
      double a = 0.0;
      int c = 0;
      for (int k = 0; k < SEG; ++k) {
        a += acc[s][part * SEG + k];
        c += cnt[s][part * SEG + k];
      }
      racc[s][part] = a;
      rcnt[s][part] = c;
    }
    __syncthreads();
    if (tid < NLEV) {
      double a = 0.0;
      int c = 0;
      for (int part = 0; part < KM_PARTS; ++part) {
        a += racc[tid][part];
        c += rcnt[tid][part];
      }
      if (c > 0) t[tid] = (double)(float)(a / (double)c);  // __ddiv_rn, then fp32 rounding
    }
  }
  __syncthreads();
  if (tid < NLEV) trow[tid] = (float)t[tid];
}

template <int NLEV>
ganq_status_t launch_kmeans_t(const float* W, int64_t m, int64_t n, int iters, float* T, cudaStream_t st) {
  kmeans_kernel<NLEV><<<(unsigned)m, KM_THREADS, 0, st>>>(W, n, iters, T);
  GANQ_LAUNCH_CHECK("kmeans_kernel");
  return GANQ_OK;
}

}  // namespace

ganq_status_t launch_kmeans_codebook(const float* W, int64_t m, int64_t n, int nlev, int iters, float* T,
                                     cudaStream_t st) {
  ganq_status_t s;
  if ((s = launch_init_codebook(W, m, n, nlev, T, st))) return s;
  if (iters == 0) return GANQ_OK;
  switch (nlev) {
    case 2: return launch_kmeans_t<2>(W, m, n, iters, T, st);
    case 4: return launch_kmeans_t<4>(W, m, n, iters, T, st);
    case 8: return launch_kmeans_t<8>(W, m, n, iters, T, st);
    case 16: return launch_kmeans_t<16>(W, m, n, iters, T, st);
    default: return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
