// gemm_tc.cu -- fp32-class contraction C = A * B^T on the tensor cores (tcgen05 kind::tf32, x3):
//   W H  (the W_i H S_i^T factor of Eq. 6; once per layer)  and
//   E H  (the objective, Eq. 8),
// with A (M x K) and B (N x K) both K-major (H is symmetric, so its rows serve as B).
//
// Split precision: every operand is pre-split into hi = tf32(x) and lo = x - hi (both exact
// fp32), and three MMAs per k-step accumulate lo*hi + hi*lo + hi*hi (error ~2^-22 relative
// per product, reading R-15).  Tensor-core fp32 accumulation truncates, so a chunk of
// 256 k (96 MMAs) is accumulated per TMEM buffer and folded by the epilogue into a
// round-to-nearest fp32 running sum, also in TMEM; C is written once per tile.
// 128 x 128 tiles, 32-wide k stages of 4 operand tiles (64 KB, SWIZZLE_128B, 3 deep).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;       // BK fp32 = 128 bytes: one swizzle row
constexpr int STAGES = 3;
constexpr int TILE = 128 * BK * 4;               // 16 KB
constexpr int STAGE_BYTES = 4 * TILE;            // A hi, A lo, B hi, B lo
constexpr int CHUNK_STAGES = 8;                  // 256 k per TMEM accumulation chain
constexpr int THREADS = 192;
constexpr uint32_t IDESC = umma_idesc(/*tf32*/ 2, 0, 0, BM, BN);

__global__ void __launch_bounds__(THREADS, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                   const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                   int64_t M, int64_t N, int64_t K, float* __restrict__ C) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(tiles + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nks = (int)((K + BK - 1) / BK);
  const int nchunks = (nks + CHUNK_STAGES - 1) / CHUNK_STAGES;

  if (threadIdx.x == 0) {
    prefetch_tmap(&mAhi);
    prefetch_tmap(&mAlo);
    prefetch_tmap(&mBhi);
    prefetch_tmap(&mBlo);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // [0,128),[128,256): chunk buffers; [256,384): running sum

  if (warp == 0) {
    if (lane == 0) {
      for (int ks = 0; ks < nks; ++ks) {
        const int s = ks % STAGES;
        mbar_wait(&empty[s], ((ks / STAGES) & 1) ^ 1);
        uint8_t* st = tiles + s * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(st, &mAhi, &full[s], ks * BK, m0);
        tma_load_2d(st + TILE, &mAlo, &full[s], ks * BK, m0);
        tma_load_2d(st + 2 * TILE, &mBhi, &full[s], ks * BK, n0);
        tma_load_2d(st + 3 * TILE, &mBlo, &full[s], ks * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int ks = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        mbar_wait(&tempty[buf], ((c >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        const int kend = min(nks, (c + 1) * CHUNK_STAGES);
        bool first = true;
        for (; ks < kend; ++ks) {
          const int s = ks % STAGES;
          mbar_wait(&full[s], (ks / STAGES) & 1);
          tc_fence_after();
          const uint32_t st = smem_u32(tiles + s * STAGE_BYTES);
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {  // lo*hi, hi*lo, hi*hi
            const uint32_t a = st + (pass == 0 ? TILE : 0);
            const uint32_t b = st + 2 * TILE + (pass == 1 ? TILE : 0);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              mma_tf32(d, umma_desc_sw128(a + kk * 32, 16, 1024), umma_desc_sw128(b + kk * 32, 16, 1024),
                       IDESC, (first && pass == 0 && kk == 0) ? 0u : 1u);
            }
          }
          first = false;
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    // epilogue: fold each chunk into the running sum; write C at the end
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lb = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      mbar_wait(&tfull[buf], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int g = 0; g < BN / 16; ++g) {
        uint32_t v[16], r[16];
        tmem_ld16(lb + buf * BN + g * 16, v);
        if (c > 0) tmem_ld16(lb + 2 * BN + g * 16, r);
        tmem_ld_wait();
        if (c > 0) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            v[q] = __float_as_uint(__fadd_rn(__uint_as_float(r[q]), __uint_as_float(v[q])));
        }
        tmem_st16(lb + 2 * BN + g * 16, v);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
    tc_fence_after();
    const int64_t gm = m0 + row;
#pragma unroll 1
    for (int g = 0; g < BN / 16; ++g) {
      uint32_t v[16];
      tmem_ld16(lb + 2 * BN + g * 16, v);
      tmem_ld_wait();
      if (gm < M) {
        float* crow = C + gm * N + n0 + g * 16;
        if (n0 + g * 16 + 16 <= N && (reinterpret_cast<uintptr_t>(crow) & 15) == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            reinterpret_cast<float4*>(crow)[q] =
                make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                            __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (n0 + g * 16 + q < N) crow[q] = __uint_as_float(v[q]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// hi = tf32(x) (round to nearest, ties away), lo = x - hi (exact); pitched rows (pitch kp).
__global__ void split_tf32_kernel(const float* __restrict__ X, int64_t rows, int64_t K, int64_t kp,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = rows * kp;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / kp, k = idx % kp;
    float h = 0.0f, l = 0.0f;
    if (k < K) {
      const float x = X[r * K + k];
      uint32_t hb;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
      h = __uint_as_float(hb);
      l = __fsub_rn(x, h);
    }
    hi[idx] = h;
    lo[idx] = l;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const float* base, int64_t K, int64_t rows, int64_t kp) {
  auto encode = encode_fn();
  if (!encode) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kp * 4};
  cuuint32_t box[2] = {BK, 128};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int64_t gemm_pitch(int64_t K) { return (K + 3) / 4 * 4; }

ganq_status_t launch_split_tf32(const float* X, int64_t rows, int64_t K, float* hi, float* lo,
                                cudaStream_t st) {
  split_tf32_kernel<<<1184, 256, 0, st>>>(X, rows, K, gemm_pitch(K), hi, lo);
  GANQ_LAUNCH_CHECK("split_tf32_kernel");
  return GANQ_OK;
}

// C (M x N) = A * B^T with A = (Ahi, Alo) M x K and B = (Bhi, Blo) N x K, pitch gemm_pitch(K).
ganq_status_t launch_gemm_tf32x3(const float* Ahi, const float* Alo, const float* Bhi, const float* Blo,
                                 int64_t M, int64_t N, int64_t K, float* C, cudaStream_t st) {
  const int64_t kp = gemm_pitch(K);
  CUtensorMap a0, a1, b0, b1;
  if (!make_map(&a0, Ahi, K, M, kp) || !make_map(&a1, Alo, K, M, kp) || !make_map(&b0, Bhi, K, N, kp) ||
      !make_map(&b1, Blo, K, N, kp)) {
    set_error(GANQ_ERR_CUDA, "gemm_tf32x3: tensor map encoding failed");
    return GANQ_ERR_CUDA;
  }
  const size_t smem = 1024 + STAGES * STAGE_BYTES + 256;
  GANQ_CUDA_TRY(cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  gemm_tf32x3_kernel<<<grid, THREADS, smem, st>>>(a0, a1, b0, b1, M, N, K, C);
  GANQ_LAUNCH_CHECK("gemm_tf32x3_kernel");
  return GANQ_OK;
}

}  // namespace ganq
