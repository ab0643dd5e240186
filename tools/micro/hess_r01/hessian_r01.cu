// hessian.cu -- H = X X^T (Algorithm 1) on the 5th-gen tensor cores.
//
// X is token-major (p x n bf16).  H_ij = sum_t X[t][i] X[t][j] is a SYRK whose
// contraction runs over the outer (row) dimension of X, so both UMMA operands
// are MN-major: TMA loads boxes of 64 channels x 64 tokens with 128-byte
// swizzle, which is exactly the canonical MN-major SW128 UMMA layout
// (8-token groups 1024 B apart = SBO, 64-channel blocks one box apart = LBO).
//
// Tiling: one CTA owns a 128 (i) x 256 (j) output tile that touches the lower
// triangle and loops over all token chunks of 8192 tokens.  A
// chunk accumulates in fp32 in TMEM columns [0, 256) (bf16 products are exact in
// fp32; the tensor-core adds truncate, so chains are kept to one chunk).  The
// epilogue folds each chunk into a round-to-nearest fp32 running sum kept in TMEM
// columns [256, 512) (tcgen05.ld + add + tcgen05.st) and writes the tile to the
// fp64 H once, at the end (reading R-12): no per-chunk read-modify-write of H.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (+TMEM owner), 2..5 = epilogue
// (one TMEM lane quarter each).  A final kernel mirrors the strict lower triangle
// onto the upper one, so H is exactly symmetric.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int BM = 128;        // i rows per tile (UMMA M)
constexpr int BN = 256;        // j cols per tile (UMMA N)
constexpr int BK = 64;         // tokens per pipeline stage
constexpr int STAGES = 4;
constexpr int BOX = 64;        // channels per TMA box (128 B of bf16)
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int THREADS = 192;
constexpr uint32_t IDESC = umma_idesc(/*bf16*/ 1, /*A MN*/ 1, /*B MN*/ 1, BM, BN);

__global__ void __launch_bounds__(THREADS, 1)
hessian_syrk_kernel(const __grid_constant__ CUtensorMap tmap, int64_t p, int64_t n,
                    double* __restrict__ H, int accumulate) {
  // grid = (TJ, TI); tiles entirely above the diagonal exit before any setup.
  const int i0 = blockIdx.y * BM;
  const int j0 = blockIdx.x * BN;
  if (j0 > i0 + BM - 1) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (p + 8192 - 1) / 8192;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t kb = 0;
      for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t t0 = c * 8192;
        const int64_t t1 = min(p, t0 + 8192);
        for (int64_t t = t0; t < t1; t += BK, ++kb) {
          const uint32_t s = kb % STAGES;
          mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
          uint8_t* a = smem + s * STAGE_BYTES;
          uint8_t* b = a + A_BYTES;
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll
          for (int q = 0; q < BM / BOX; ++q)
            tma_load_2d(a + q * (BK * 128), &tmap, &full[s], i0 + q * BOX, (int)t);
#pragma unroll
          for (int q = 0; q < BN / BOX; ++q)
            tma_load_2d(b + q * (BK * 128), &tmap, &full[s], j0 + q * BOX, (int)t);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      uint32_t kb = 0;
      for (int64_t c = 0; c < nchunks; ++c) {
        const uint32_t buf = 0;
        mbar_wait(&tempty[0], ((uint32_t)c & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base;
        const int64_t t0 = c * 8192;
        const int64_t t1 = min(p, t0 + 8192);
        bool first = true;
        for (int64_t t = t0; t < t1; t += BK, ++kb) {
          const uint32_t s = kb % STAGES;
          mbar_wait(&full[s], (kb / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // 16 tokens = 16 rows of 128 B inside every 64-channel box.
            const uint64_t ad = umma_desc_sw128(a_addr + kk * 2048, BK * 128, 1024);
            const uint64_t bd = umma_desc_sw128(b_addr + kk * 2048, BK * 128, 1024);
            mma_f16(d_tmem, ad, bd, IDESC, (first && kk == 0) ? 0u : 1u);
          }
          first = false;
          mma_commit(&empty[s]);  // frees the smem stage when these MMAs retire
        }
        mma_commit(&tfull[buf]);  // chunk accumulator ready for the epilogue
        (void)buf;
      }
    }
  } else {
    // ---------------- epilogue: fold chunks into the TMEM fp32 running sum, write H once
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, +32) are accessible to this warp
    const int row = quarter * 32 + lane;
    const int64_t gi = (int64_t)i0 + row;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    for (int64_t c = 0; c < nchunks; ++c) {
      mbar_wait(&tfull[0], (uint32_t)c & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cg = 0; cg < BN / 16; ++cg) {
        uint32_t v[16], r[16];
        tmem_ld16(lane_base + cg * 16, v);
        if (c > 0) tmem_ld16(lane_base + BN + cg * 16, r);
        tmem_ld_wait();
        if (c > 0) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            v[q] = __float_as_uint(__fadd_rn(__uint_as_float(r[q]), __uint_as_float(v[q])));
        }
        tmem_st16(lane_base + BN + cg * 16, v);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
    }
    tc_fence_after();
#pragma unroll 1
    for (int cg = 0; cg < BN / 16; ++cg) {
      uint32_t v[16];
      tmem_ld16(lane_base + BN + cg * 16, v);
      tmem_ld_wait();
      if (gi < n) {
        double* hrow = H + gi * n;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t gj = (int64_t)j0 + cg * 16 + q;
          if (gj < n && gj <= gi) {
            const double val = (double)__uint_as_float(v[q]);
            hrow[gj] = accumulate ? hrow[gj] + val : val;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

// H[j][i] = H[i][j] for i > j (tiled transpose through shared memory).
__global__ void mirror_lower_kernel(double* __restrict__ H, int64_t n) {
  __shared__ double tile[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;  // source tile rows bi, cols bj, bi >= bj
  if (bj > bi) return;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bi * 32 + r, j = bj * 32 + tx;
    if (i < n && j < n) tile[r][tx] = H[i * n + j];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bj * 32 + r, j = bi * 32 + tx;  // destination (i, j) = source (j, i)
    if (i < n && j < n && j > i) H[i * n + j] = tile[tx][r];
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

}  // namespace

ganq_status_t launch_hessian(const uint16_t* X, int64_t p, int64_t n, double* H, int accumulate,
                             cudaStream_t st) {
  if (n % 8 != 0) {
    set_error(GANQ_ERR_UNSUPPORTED, "ganq_hessian: n = %lld must be a multiple of 8", (long long)n);
    return GANQ_ERR_UNSUPPORTED;
  }
  if (n > (1 << 30) || p > ((int64_t)1 << 31) - 1) {
    set_error(GANQ_ERR_UNSUPPORTED, "ganq_hessian: p or n too large for 32-bit TMA coordinates");
    return GANQ_ERR_UNSUPPORTED;
  }
  if (reinterpret_cast<uintptr_t>(X) % 16 != 0) {
    set_error(GANQ_ERR_INVALID_ARG, "ganq_hessian: X must be 16-byte aligned");
    return GANQ_ERR_INVALID_ARG;
  }
  auto encode = get_encode_fn();
  if (!encode) {
    set_error(GANQ_ERR_CUDA, "ganq_hessian: cuTensorMapEncodeTiled unavailable");
    return GANQ_ERR_CUDA;
  }
  CUtensorMap tmap;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)p};
  cuuint64_t strides[1] = {(cuuint64_t)n * 2};
  cuuint32_t box[2] = {BOX, BK};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)X, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(GANQ_ERR_CUDA, "ganq_hessian: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GANQ_ERR_CUDA;
  }
  const int TI = (int)((n + BM - 1) / BM);
  const int TJ = (int)((n + BN - 1) / BN);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(hessian_syrk_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  hessian_syrk_kernel<<<dim3(TJ, TI), THREADS, SMEM_BYTES, st>>>(tmap, p, n, H, accumulate);
  GANQ_LAUNCH_CHECK("hessian_syrk_kernel");
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  mirror_lower_kernel<<<grid, dim3(32, 8), 0, st>>>(H, n);
  GANQ_LAUNCH_CHECK("mirror_lower_kernel");
  return GANQ_OK;
}

}  // namespace ganq
