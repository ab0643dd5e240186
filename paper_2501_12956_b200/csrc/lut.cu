// lut.cu -- NEXT-1, the deployment side of GANQ: N-bit packing of the codes and the LUT-based
// mixed-precision GEMM of Fig. 1a right, W~_ij = t_{i, Q_ij}, storage as in
// Table 1 (fp16 codebook, N bits per code).
//
// lut_gemm: one warp per row of W~ (grid-stride).  A row's packed codes are read once from
// HBM (coalesced: lane l takes the 8 codes [256 c + 8 l, +8) of chunk c, N bytes); the row's
// 2^N codebook entries sit as fp32 in 16 distinct shared-memory banks (a lookup is one
// conflict-free LDS); X (p x n fp16, L2-resident) is staged once per CTA in shared memory.
// Each lane accumulates its codes in ascending j in fp32, then a fixed butterfly over the
// warp: deterministic.  HBM-bound: n N / 8 + 2^{N+1} bytes per row.
#include <cuda_fp16.h>
#include <stdlib.h>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int LUT_WARPS = 8;
constexpr int LUT_PMAX = 8;  // tokens per launch (decode)
constexpr int LUT_CH = 16;   // chunks of 256 codes whose loads are issued together

__global__ void pack_kernel(const uint8_t* __restrict__ Q, int64_t m, int64_t n, int N,
                            uint8_t* __restrict__ P) {
  const int64_t rb = (n * N + 7) / 8, groups = (n + 7) / 8;
  const uint32_t mask = (1u << N) - 1u;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * groups;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / groups, g = idx % groups;
    const int64_t k0 = 8 * g;
    const int cnt = (int)min((int64_t)8, n - k0);
    uint64_t v = 0;
    for (int k = 0; k < cnt; ++k) v |= (uint64_t)(Q[i * n + k0 + k] & mask) << (k * N);
    const int nbytes = (cnt * N + 7) / 8;  // 8 codes = N whole bytes
    uint8_t* dst = P + i * rb + g * N;
    for (int b = 0; b < nbytes; ++b) dst[b] = (uint8_t)(v >> (8 * b));
  }
}

__global__ void codebook_f16_kernel(const float* __restrict__ T, int64_t total, __half* __restrict__ T16) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    T16[idx] = __float2half_rn(T[idx]);
}

template <int N, int PT>
__global__ void __launch_bounds__(32 * LUT_WARPS)
lut_gemm_kernel(const uint8_t* __restrict__ P, const __half* __restrict__ T16, const __half* __restrict__ X,
                int64_t m, int64_t n, int64_t p, float* __restrict__ Y) {
  extern __shared__ __align__(16) uint8_t lut_smem[];
  constexpr int NL = 1 << N;
  float* sT = reinterpret_cast<float*>(lut_smem);              // [LUT_WARPS][NL]
  __half* sX = reinterpret_cast<__half*>(sT + LUT_WARPS * NL);  // [PT][npad]
  const int64_t npad = (n + 255) / 256 * 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // p = 1 reads its activations straight from global memory (8 KB, L1/L2-resident), issued
  // with the codes; p > 1 stages X in shared memory once per CTA (16-byte loads when aligned)
  const bool xvec = (n & 7) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  if constexpr (PT > 1) {
    if (xvec) {
      for (int64_t e = threadIdx.x; e < PT * npad / 8; e += blockDim.x) {
        const int64_t t = (8 * e) / npad, j = (8 * e) % npad;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (t < p && j < n) v = __ldg(reinterpret_cast<const uint4*>(X + t * n + j));
        *reinterpret_cast<uint4*>(sX + 8 * e) = v;
      }
    } else {
      for (int64_t e = threadIdx.x; e < PT * npad; e += blockDim.x) {
        const int64_t t = e / npad, j = e % npad;
        sX[e] = (t < p && j < n) ? X[t * n + j] : __float2half_rn(0.0f);
      }
    }
    __syncthreads();
  }
  const int64_t rb = (n * N + 7) / 8;
  const int64_t chunks = npad / 256;
  const uint32_t mask = NL - 1;
  for (int64_t row = (int64_t)blockIdx.x * LUT_WARPS + warp; row < m; row += (int64_t)gridDim.x * LUT_WARPS) {
    for (int e = lane; e < NL; e += 32) sT[warp * NL + e] = __half2float(T16[row * NL + e]);
    __syncwarp();
    const uint8_t* prow = P + row * rb;
    float acc[PT];
#pragma unroll
    for (int t = 0; t < PT; ++t) acc[t] = 0.0f;
    // the codes of LUT_CH chunks are loaded first (independent loads in flight), then used
    auto load_bits = [&](int64_t c) -> uint64_t {
      const int64_t j0 = 256 * c + 8 * lane;  // this lane's first code in the chunk
      const int64_t b0 = j0 * N / 8;          // its first byte (8 codes = N whole bytes)
      uint64_t bits = 0;
      if (j0 + 8 <= n) {
        if constexpr (N == 4) {
          bits = (reinterpret_cast<uintptr_t>(prow + b0) & 3) == 0
                     ? __ldg(reinterpret_cast<const uint32_t*>(prow + b0))
                     : (uint64_t)prow[b0] | ((uint64_t)prow[b0 + 1] << 8) | ((uint64_t)prow[b0 + 2] << 16) |
                           ((uint64_t)prow[b0 + 3] << 24);
        } else {
#pragma unroll
          for (int b = 0; b < N; ++b) bits |= (uint64_t)__ldg(prow + b0 + b) << (8 * b);
        }
      } else if (j0 < n) {
        const int64_t nb = ((n - j0) * N + 7) / 8;
        for (int b = 0; b < nb; ++b) bits |= (uint64_t)prow[b0 + b] << (8 * b);
      }
      return bits;
    };
    for (int64_t c0 = 0; c0 < chunks; c0 += LUT_CH) {
      uint64_t bits[LUT_CH];
      uint4 xg[PT == 1 ? LUT_CH : 1];
#pragma unroll
      for (int u = 0; u < LUT_CH; ++u) {
        bits[u] = (c0 + u < chunks) ? load_bits(c0 + u) : 0;
        if constexpr (PT == 1) {
          const int64_t j0 = 256 * (c0 + u) + 8 * lane;
          if (xvec && j0 + 8 <= n) {
            xg[u] = __ldg(reinterpret_cast<const uint4*>(X + j0));
          } else {
            __half h[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) h[k] = (j0 + k < n) ? X[j0 + k] : __float2half_rn(0.0f);
            xg[u] = *reinterpret_cast<const uint4*>(h);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < LUT_CH; ++u) {
        if (c0 + u >= chunks) break;
        const int64_t j0 = 256 * (c0 + u) + 8 * lane;
        float w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          w[k] = (j0 + k < n) ? sT[warp * NL + ((bits[u] >> (k * N)) & mask)] : 0.0f;
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          const uint4 xv = (PT == 1) ? xg[u] : *reinterpret_cast<const uint4*>(sX + t * npad + j0);  // 8 halfs
          const __half2* xh = reinterpret_cast<const __half2*>(&xv);
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const float2 xf = __half22float2(xh[k2]);
            acc[t] = fmaf(w[2 * k2], xf.x, acc[t]);
            acc[t] = fmaf(w[2 * k2 + 1], xf.y, acc[t]);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < PT; ++t)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < PT; ++t)
        if (t < p) Y[t * m + row] = acc[t];
    }
    __syncwarp();
  }
}

// Fast path for the common shape: N = 4, n a multiple of 256 (whole chunks, 4-byte aligned code
// words), X 16-byte aligned.  fmaf into fp32 in ascending j per lane, split over NA accumulators
// by the code's position in its word (4 for one token, 2 for two), added in a fixed order, then
// the butterfly; 4 CTAs per SM (64 registers) so that one launch covers m = 4096 rows in one wave.
template <int PT>
__global__ void __launch_bounds__(32 * LUT_WARPS, PT <= 2 ? 4 : 2)
lut4_gemm_kernel(const uint8_t* __restrict__ P, const __half* __restrict__ T16, const __half* __restrict__ X,
                 int m, int n, int p, float* __restrict__ Y) {
  __shared__ __align__(512) float sT[LUT_WARPS * 16];
  extern __shared__ __align__(16) float sXf[];  // [PT][n] fp32 (converted once per CTA)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks0 = n >> 8, rb0 = n >> 1;
  // the first row's codes and codebook entry are requested before X is staged (overlap)
  uint32_t bn[LUT_CH];
  float tn = 0.0f;
  auto prefetch = [&](int r) {
    const uint32_t* pr = reinterpret_cast<const uint32_t*>(P + (int64_t)r * rb0);
#pragma unroll
    for (int u = 0; u < LUT_CH; ++u) bn[u] = (u < chunks0) ? __ldg(pr + 32 * u + lane) : 0u;  // 128 B per chunk
    tn = __half2float(T16[(int64_t)r * 16 + (lane & 15)]);
  };
  if (blockIdx.x * LUT_WARPS + warp < m) prefetch(blockIdx.x * LUT_WARPS + warp);
  for (int e = threadIdx.x; e < PT * n / 8; e += blockDim.x) {
    const int t = (8 * e) / n, j = (8 * e) % n;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t < p) v = __ldg(reinterpret_cast<const uint4*>(X + (int64_t)t * n + j));
    const __half2* h = reinterpret_cast<const __half2*>(&v);
    float4 f0, f1;
    f0.x = __low2float(h[0]); f0.y = __high2float(h[0]); f0.z = __low2float(h[1]); f0.w = __high2float(h[1]);
    f1.x = __low2float(h[2]); f1.y = __high2float(h[2]); f1.z = __low2float(h[3]); f1.w = __high2float(h[3]);
    reinterpret_cast<float4*>(sXf + 8 * e)[0] = f0;
    reinterpret_cast<float4*>(sXf + 8 * e)[1] = f1;
  }
  __syncthreads();
  const int chunks = n >> 8, rb = n >> 1;
  // shared address of this warp's 16 fp32 entries (64-byte aligned), OR-ed with (code * 4): the
  // address of a lookup is one LOP3 of the shifted code word
  const uint32_t tsh = smem_u32(sT) + (uint32_t)warp * 64u;
  // one row per warp when m <= the resident warps (the launch is sized for it)
  const int stride = gridDim.x * LUT_WARPS;
  int row = blockIdx.x * LUT_WARPS + warp;
  for (bool first = true; row < m; row += stride, first = false) {
    // (the first row's codes and codebook entry were requested before X was staged; later rows
    // -- only when m exceeds the resident warps -- load theirs here)
    if (!first) prefetch(row);
    const uint32_t* b0 = bn;
    if (lane < 16) sT[warp * 16 + lane] = tn;
    __syncwarp();
    const uint32_t* prow = reinterpret_cast<const uint32_t*>(P + (int64_t)row * rb);
    // NA independent accumulators per token (code k of a word -> accumulator k % NA): short
    // dependent FMA chains, then a fixed-order combine and the butterfly
    constexpr int NA = PT == 1 ? 4 : (PT == 2 ? 2 : 1);
    float acc[PT][NA];
#pragma unroll
    for (int t = 0; t < PT; ++t)
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[t][a] = 0.0f;
    for (int c0 = 0; c0 < chunks; c0 += LUT_CH) {
      uint32_t b[LUT_CH];
#pragma unroll
      for (int u = 0; u < LUT_CH; ++u)
        b[u] = (c0 == 0) ? b0[u] : ((c0 + u < chunks) ? __ldg(prow + 32 * (c0 + u) + lane) : 0u);
#pragma unroll
      for (int u = 0; u < LUT_CH; ++u) {
        if (c0 + u >= chunks) break;
        float w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t sh = (k == 0 ? (b[u] << 2) : (b[u] >> (4 * k - 2)));
          uint32_t addr;
          asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(addr) : "r"(sh), "r"(0x3Cu), "r"(tsh));  // (sh & 0x3C) | tsh
          // (memory clobber: ordered after this row's table store and before the next one's)
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(w[k]) : "r"(addr) : "memory");
        }
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          const float4* xp = reinterpret_cast<const float4*>(sXf + t * n + 256 * (c0 + u) + 8 * lane);
          const float4 x0 = xp[0], x1 = xp[1];
          const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[t][k % NA] = fmaf(w[k], xv[k], acc[t][k % NA]);
        }
      }
    }
    float accs[PT];
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      accs[t] = acc[t][0];
#pragma unroll
      for (int a = 1; a < NA; ++a) accs[t] = __fadd_rn(accs[t], acc[t][a]);
    }
#pragma unroll
    for (int t = 0; t < PT; ++t)
#pragma unroll
      for (int o = 16; o; o >>= 1) accs[t] += __shfl_xor_sync(0xffffffffu, accs[t], o);
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < PT; ++t)
        if (t < p) Y[(int64_t)t * m + row] = accs[t];
    }
    __syncwarp();
  }
}

// Fast path for any N and n a multiple of 256: a chunk of 256 codes is 32 N bytes = 8 N words;
// lanes < 8 N load one word each (coalesced), then every lane gathers its 8 N-bit window (codes
// [8 l, 8 l + 8) of the chunk) with shuffles and a funnel shift.  Lookup and summation as in
// lut4_gemm_kernel (same order: a lane's codes ascending, fmaf in fp32, then the butterfly).
template <int N, int PT>
__global__ void __launch_bounds__(32 * LUT_WARPS)
lutn_gemm_kernel(const uint8_t* __restrict__ P, const __half* __restrict__ T16, const __half* __restrict__ X,
                 int m, int n, int p, float* __restrict__ Y) {
  constexpr int NL = 1 << N;
  constexpr int WPC = 8 * N;  // words per chunk
  __shared__ __align__(1024) float sT[LUT_WARPS * NL];
  extern __shared__ __align__(16) float sXf[];  // [PT][n] fp32
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = n >> 8;
  const int64_t rbw = (int64_t)n * N / 32;  // row length in words (n % 256 == 0)
  uint32_t wn[2][LUT_CH];                    // prefetched words (lanes < WPC; two per lane if N > 4)
  auto prefetch = [&](int r) {
    const uint32_t* pr = reinterpret_cast<const uint32_t*>(P) + (int64_t)r * rbw;
#pragma unroll
    for (int u = 0; u < LUT_CH; ++u) {
      wn[0][u] = (u < chunks && lane < WPC) ? __ldg(pr + WPC * u + lane) : 0u;
      wn[1][u] = (N > 4 && u < chunks && lane + 32 < WPC) ? __ldg(pr + WPC * u + lane + 32) : 0u;
    }
  };
  if (blockIdx.x * LUT_WARPS + warp < m) prefetch(blockIdx.x * LUT_WARPS + warp);
  for (int e = threadIdx.x; e < PT * n / 8; e += blockDim.x) {
    const int t = (8 * e) / n, j = (8 * e) % n;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t < p) v = __ldg(reinterpret_cast<const uint4*>(X + (int64_t)t * n + j));
    const __half2* h = reinterpret_cast<const __half2*>(&v);
    float4 f0, f1;
    f0.x = __low2float(h[0]); f0.y = __high2float(h[0]); f0.z = __low2float(h[1]); f0.w = __high2float(h[1]);
    f1.x = __low2float(h[2]); f1.y = __high2float(h[2]); f1.z = __low2float(h[3]); f1.w = __high2float(h[3]);
    reinterpret_cast<float4*>(sXf + 8 * e)[0] = f0;
    reinterpret_cast<float4*>(sXf + 8 * e)[1] = f1;
  }
  __syncthreads();
  const uint32_t tsh = smem_u32(sT) + (uint32_t)(warp * NL * 4);  // aligned to NL * 4 bytes
  const int bit0 = 8 * N * lane;                                  // first bit of this lane in a chunk
  const int wsrc = bit0 >> 5, sh0 = bit0 & 31;
  const int stride = gridDim.x * LUT_WARPS;
  for (int row = blockIdx.x * LUT_WARPS + warp; row < m; row += stride) {
    uint32_t w0[LUT_CH], w1[LUT_CH];
#pragma unroll
    for (int u = 0; u < LUT_CH; ++u) { w0[u] = wn[0][u]; w1[u] = wn[1][u]; }
    for (int e = lane; e < NL; e += 32) sT[warp * NL + e] = __half2float(T16[(int64_t)row * NL + e]);
    if (row + stride < m) prefetch(row + stride);
    __syncwarp();
    const uint32_t* prow = reinterpret_cast<const uint32_t*>(P) + (int64_t)row * rbw;
    float acc[PT];
#pragma unroll
    for (int t = 0; t < PT; ++t) acc[t] = 0.0f;
    for (int c0 = 0; c0 < chunks; c0 += LUT_CH) {
      uint32_t a0[LUT_CH], a1[LUT_CH];
#pragma unroll
      for (int u = 0; u < LUT_CH; ++u) {
        const bool in = c0 + u < chunks;
        a0[u] = (c0 == 0) ? w0[u] : ((in && lane < WPC) ? __ldg(prow + WPC * (c0 + u) + lane) : 0u);
        a1[u] = (c0 == 0) ? w1[u] : ((N > 4 && in && lane + 32 < WPC) ? __ldg(prow + WPC * (c0 + u) + lane + 32) : 0u);
      }
#pragma unroll
      for (int u = 0; u < LUT_CH; ++u) {
        if (c0 + u >= chunks) break;
        // gather words wsrc, wsrc + 1, wsrc + 2 of the chunk (word q lives in lane q % 32, set q / 32)
        auto word = [&](int q) {
          const uint32_t lo = __shfl_sync(0xffffffffu, a0[u], q & 31);
          if constexpr (N > 4) {
            const uint32_t hi = __shfl_sync(0xffffffffu, a1[u], q & 31);
            return q < 32 ? lo : hi;
          }
          return lo;
        };
        const uint32_t x0 = word(wsrc), x1 = word(wsrc + 1);
        uint64_t bits = (((uint64_t)x1 << 32) | x0) >> sh0;
        if constexpr (N > 4) {  // the shuffle runs in every lane (full-mask), the select afterwards
          const uint64_t x2 = word(wsrc + 2);
          bits |= (sh0 > 0) ? (x2 << (64 - sh0)) : 0ull;
        }
        float w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // (code k) * 4 sits at bits [N k - 2, ...): shift right by N k - 2, or left when N k < 2
          const uint32_t shv = (N * k >= 2) ? (uint32_t)(bits >> (N * k - 2)) : (uint32_t)(bits << (2 - N * k));
          uint32_t addr;
          asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(addr) : "r"(shv), "r"((uint32_t)(NL - 1) << 2), "r"(tsh));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(w[k]) : "r"(addr) : "memory");
        }
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          const float4* xp = reinterpret_cast<const float4*>(sXf + t * n + 256 * (c0 + u) + 8 * lane);
          const float4 xa = xp[0], xb = xp[1];
          acc[t] = fmaf(w[0], xa.x, acc[t]);
          acc[t] = fmaf(w[1], xa.y, acc[t]);
          acc[t] = fmaf(w[2], xa.z, acc[t]);
          acc[t] = fmaf(w[3], xa.w, acc[t]);
          acc[t] = fmaf(w[4], xb.x, acc[t]);
          acc[t] = fmaf(w[5], xb.y, acc[t]);
          acc[t] = fmaf(w[6], xb.z, acc[t]);
          acc[t] = fmaf(w[7], xb.w, acc[t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < PT; ++t)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < PT; ++t)
        if (t < p) Y[(int64_t)t * m + row] = acc[t];
    }
    __syncwarp();
  }
}

template <int N, int PT>
ganq_status_t launch_lutn_t(const uint8_t* P, const __half* T16, const __half* X, int64_t m, int64_t n, int64_t p,
                            float* Y, cudaStream_t st) {
  const size_t smem = (size_t)PT * n * sizeof(float);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(lutn_gemm_kernel<N, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lutn_gemm_kernel<N, PT>, 32 * LUT_WARPS, smem);
  const int64_t want = (m + LUT_WARPS - 1) / LUT_WARPS;
  const unsigned grid = (unsigned)min(want, (int64_t)sms * (per_sm > 0 ? per_sm : 1));
  lutn_gemm_kernel<N, PT><<<grid, 32 * LUT_WARPS, smem, st>>>(P, T16, X, (int)m, (int)n, (int)p, Y);  // persistent
  GANQ_LAUNCH_CHECK("lutn_gemm_kernel");
  return GANQ_OK;
}

template <int PT>
ganq_status_t launch_lut4_t(const uint8_t* P, const __half* T16, const __half* X, int64_t m, int64_t n, int64_t p,
                            float* Y, cudaStream_t st) {
  const size_t smem = (size_t)PT * n * sizeof(float);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(lut4_gemm_kernel<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut4_gemm_kernel<PT>, 32 * LUT_WARPS, smem);
  static const int cap = getenv("GANQ_LUT_CTAS_PER_SM") ? atoi(getenv("GANQ_LUT_CTAS_PER_SM")) : 0;
  if (cap > 0 && cap < per_sm) per_sm = cap;
  const int64_t want = (m + LUT_WARPS - 1) / LUT_WARPS;
  const unsigned grid = (unsigned)min(want, (int64_t)sms * (per_sm > 0 ? per_sm : 1));
  lut4_gemm_kernel<PT><<<grid, 32 * LUT_WARPS, smem, st>>>(P, T16, X, (int)m, (int)n, (int)p, Y);  // persistent
  GANQ_LAUNCH_CHECK("lut4_gemm_kernel");
  return GANQ_OK;
}

template <int N, int PT>
ganq_status_t launch_lut_t(const uint8_t* P, const __half* T16, const __half* X, int64_t m, int64_t n, int64_t p,
                           float* Y, cudaStream_t st) {
  const int64_t npad = (n + 255) / 256 * 256;
  const size_t smem = (size_t)LUT_WARPS * (1 << N) * sizeof(float) + (PT > 1 ? (size_t)PT * npad * sizeof(__half) : 0);
  if (smem > 227 * 1024) {
    set_error(GANQ_ERR_UNSUPPORTED, "lut_gemm: n = %lld too large for the shared-memory staging of X",
              (long long)n);
    return GANQ_ERR_UNSUPPORTED;
  }
  GANQ_CUDA_TRY(cudaFuncSetAttribute(lut_gemm_kernel<N, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lut_gemm_kernel<N, PT>, 32 * LUT_WARPS, smem);
  const int64_t want = (m + LUT_WARPS - 1) / LUT_WARPS;
  const unsigned grid = (unsigned)min(want, (int64_t)sms * (per_sm > 0 ? per_sm : 1));
  lut_gemm_kernel<N, PT><<<grid, 32 * LUT_WARPS, smem, st>>>(P, T16, X, m, n, p, Y);
  GANQ_LAUNCH_CHECK("lut_gemm_kernel");
  return GANQ_OK;
}

template <int N>
ganq_status_t launch_lut_n(const uint8_t* P, const __half* T16, const __half* X, int64_t m, int64_t n, int64_t p,
                           float* Y, cudaStream_t st) {
  // whole chunks (n % 256 == 0: 32 N-byte chunks, word-aligned packed rows), 16-byte aligned X,
  // and X of the batch (fp32) within shared memory
  const bool whole = n % 256 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(P) & 3) == 0 && m < (1ll << 31) && n * LUT_PMAX < (1ll << 31);
  for (int64_t t0 = 0; t0 < p; t0 += LUT_PMAX) {
    const int64_t pb = min((int64_t)LUT_PMAX, p - t0);
    const int64_t ptile = pb == 1 ? 1 : pb == 2 ? 2 : pb <= 4 ? 4 : 8;
    const bool fits = (size_t)ptile * n * sizeof(float) <= 200 * 1024;
    const bool fast = N == 4 && whole && fits, fastn = N != 4 && whole && fits;
    ganq_status_t s;
    const __half* Xb = X + t0 * n;
    float* Yb = Y + t0 * m;
    if (fast) {
      if (pb == 1) s = launch_lut4_t<1>(P, T16, Xb, m, n, pb, Yb, st);
      else if (pb == 2) s = launch_lut4_t<2>(P, T16, Xb, m, n, pb, Yb, st);
      else if (pb <= 4) s = launch_lut4_t<4>(P, T16, Xb, m, n, pb, Yb, st);
      else s = launch_lut4_t<8>(P, T16, Xb, m, n, pb, Yb, st);
      if (s) return s;
      continue;
    }
    if (fastn) {
      if (pb == 1) s = launch_lutn_t<N, 1>(P, T16, Xb, m, n, pb, Yb, st);
      else if (pb == 2) s = launch_lutn_t<N, 2>(P, T16, Xb, m, n, pb, Yb, st);
      else if (pb <= 4) s = launch_lutn_t<N, 4>(P, T16, Xb, m, n, pb, Yb, st);
      else s = launch_lutn_t<N, 8>(P, T16, Xb, m, n, pb, Yb, st);
      if (s) return s;
      continue;
    }
    if (pb == 1) s = launch_lut_t<N, 1>(P, T16, Xb, m, n, pb, Yb, st);
    else if (pb == 2) s = launch_lut_t<N, 2>(P, T16, Xb, m, n, pb, Yb, st);
    else if (pb <= 4) s = launch_lut_t<N, 4>(P, T16, Xb, m, n, pb, Yb, st);
    else s = launch_lut_t<N, 8>(P, T16, Xb, m, n, pb, Yb, st);
    if (s) return s;
  }
  return GANQ_OK;
}

}  // namespace

ganq_status_t launch_pack_codes(const uint8_t* Q, int64_t m, int64_t n, int N, uint8_t* P, cudaStream_t st) {
  pack_kernel<<<1184, 256, 0, st>>>(Q, m, n, N, P);
  GANQ_LAUNCH_CHECK("pack_kernel");
  return GANQ_OK;
}

ganq_status_t launch_codebook_f16(const float* T, int64_t total, uint16_t* T16, cudaStream_t st) {
  codebook_f16_kernel<<<(unsigned)min((int64_t)1184, (total + 255) / 256), 256, 0, st>>>(
      T, total, reinterpret_cast<__half*>(T16));
  GANQ_LAUNCH_CHECK("codebook_f16_kernel");
  return GANQ_OK;
}

ganq_status_t launch_lut_gemm(const uint8_t* P, const uint16_t* T16, const uint16_t* X, int64_t m, int64_t n,
                              int64_t p, int N, float* Y, cudaStream_t st) {
  const __half* t = reinterpret_cast<const __half*>(T16);
  const __half* x = reinterpret_cast<const __half*>(X);
  switch (N) {
    case 1: return launch_lut_n<1>(P, t, x, m, n, p, Y, st);
    case 2: return launch_lut_n<2>(P, t, x, m, n, p, Y, st);
    case 3: return launch_lut_n<3>(P, t, x, m, n, p, Y, st);
    case 4: return launch_lut_n<4>(P, t, x, m, n, p, Y, st);
    case 5: return launch_lut_n<5>(P, t, x, m, n, p, Y, st);
    case 6: return launch_lut_n<6>(P, t, x, m, n, p, Y, st);
    case 7: return launch_lut_n<7>(P, t, x, m, n, p, Y, st);
    case 8: return launch_lut_n<8>(P, t, x, m, n, p, Y, st);
    default:
      set_error(GANQ_ERR_INVALID_ARG, "lut_gemm: n_bits = %d not in [1, 8]", N);
      return GANQ_ERR_INVALID_ARG;
  }
}

}  // namespace ganq
