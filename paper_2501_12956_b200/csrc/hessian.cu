// hessian.cu -- H = X X^T (Algorithm 1) on the 5th-gen tensor cores.
//
// X is token-major (p x n bf16).  H_ij = sum_t X[t][i] X[t][j] is a SYRK whose contraction runs
// over the outer (row) dimension of X, so both UMMA operands are MN-major: TMA loads boxes of 64
// channels x 64 tokens with 128-byte swizzle, which is exactly the canonical MN-major SW128 UMMA
// layout (8-token groups 1024 B apart = SBO, 64-channel blocks one box apart = LBO).
//
// Arithmetic (reading R-12):
//  * bf16 products are exact in fp32; the tensor core adds them into an fp32 TMEM accumulator.
//    Its adds truncate (~1 ulp of the accumulator per MMA of K = 16, one-sided), so a chain is
//    kept to one CHUNK of 256 tokens (16 MMAs); chunks are added into a round-to-nearest fp32
//    running sum R held in the epilogue's registers.
//  * Tokens are cut into fixed SUPER-chunks of GANQ_HESSIAN_SUPERCHUNK = 32768 tokens counted from
//    token 0 of the call.  Each super-chunk's R is stored (fp32) as a PARTIAL; a second kernel
//    rounds every partial onto the integer grid 2^(E_i + E_j - 46) and adds them in int64 --
//    exact and associative, so the result is bitwise the same for any grouping of super-chunks
//    into token shards (multi-GPU).
//  * E comes from the partials themselves: E_c = ceil(e_c / 2) + 1 with D_c = max over the
//    super-chunks of the diagonal partial P_sc[c][c] = m 2^(e_c), m in [0.5, 1) (frexp, exact).
//    Then |P_sc[i][j]| <= sqrt(P_sc[i][i] P_sc[j][j]) < 2^(E_i + E_j - 2) (Cauchy-Schwarz), i.e.
//    < 2^44 grid units per super-chunk and < 2^60 over the < 2^16 super-chunks of p < 2^31
//    tokens.  The max is order-free: ranks reduce E with MAX and get the grid of one call.
//
// Tiling: one CTA per 128 (i) x 256 (j) lower-triangle tile (1-D grid over the tile list).
// TMEM: two 256-column chunk accumulators (double-buffered: a chunk's fold overlaps the next
// chunk's MMAs).  Warp roles: 0 = TMA producer, 1 = MMA issuer (+TMEM owner), 2..9 = epilogue
// (warp w reads TMEM lane quarter w % 4 and column half (w - 2) / 4: 128 registers of R per
// thread).  Partials are [super-chunk][tile][256 j][128 i] fp32 (a warp's
// lanes -- rows -- store 128 contiguous bytes).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int BM = 128;        // i rows per CTA (the pair's UMMA M = 256)
constexpr int BN = 256;        // j cols per tile (UMMA N; each CTA of the pair stages half of B)
constexpr int BK = 64;         // tokens per pipeline stage
constexpr int STAGES = 6;
constexpr int BOX = 64;        // channels per TMA box (128 B of bf16)
constexpr int A_BYTES = BM * BK * 2;        // 16 KB: this CTA's 128 rows of A
constexpr int B_BYTES = (BN / 2) * BK * 2;  // 16 KB: this CTA's half of B
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 512 /*barriers*/;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr uint32_t IDESC = umma_idesc(/*bf16*/ 1, /*A MN*/ 1, /*B MN*/ 1, 2 * BM, BN);  // cta_group::2
constexpr int64_t SUPER = GANQ_HESSIAN_SUPERCHUNK;
constexpr int64_t CHUNK_DEFAULT = 256;  // tokens per truncating tensor-core chain (16 MMAs)
constexpr int GRID_SHIFT = 46;     // grid exponent E_i + E_j - 46
constexpr int TILE_ELEMS = BM * BN;
constexpr int E_MIN = -126;        // E of an all-zero channel

static_assert(SUPER % CHUNK_DEFAULT == 0 && CHUNK_DEFAULT % BK == 0, "chunks on stage boundaries, super-chunks on chunks");

// tile list of the lower triangle in CTA PAIRS: pair P <-> (I, J), J <= I, 256 x 256 blocks in
// row-major order; CTA c = 2 P + r owns rows [256 I + 128 r, +128) x columns [256 J, +256)
__host__ __device__ inline void pair_of(int P, int& I, int& J) {
  I = 0;
  while (P > I) P -= ++I;
  J = P;
}
__host__ __device__ inline void tile_of(int c, int& row0, int& col0) {
  int I, J;
  pair_of(c >> 1, I, J);
  row0 = 256 * I + BM * (c & 1);
  col0 = 256 * J;
}

__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
hessian_syrk_kernel(const __grid_constant__ CUtensorMap tmap, int64_t p, int64_t n, float* __restrict__ Psc,
                    int64_t CHUNK) {
  const int ntiles = gridDim.x;
  int i0, j0;
  tile_of(blockIdx.x, i0, j0);
  const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the pair's MMAs)
  const bool leader = (rank == 0);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);  // leader's counts both CTAs
  uint64_t* empty = full + STAGES;     // per CTA: the pair's MMA commit
  uint64_t* tfull = empty + STAGES;    // [2] per CTA
  uint64_t* tempty = tfull + 2;        // [2] leader's: both CTAs' epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (p + CHUNK - 1) / CHUNK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 2 * EPI_WARPS); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and TMEM exist before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: this CTA's rows of A and its half of B, every 64-token
    // stage; completion counted on the LEADER's full barrier (expecting both CTAs' bytes)
    if (lane == 0) {
      uint32_t kb = 0;
      for (int64_t t = 0; t < p; t += BK, ++kb) {
        const uint32_t s = kb % STAGES;
        mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
        uint8_t* a = smem + s * STAGE_BYTES;
        uint8_t* b = a + A_BYTES;
        if (leader) mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
#pragma unroll
        for (int q = 0; q < BM / BOX; ++q) tma_load_2d_pair(a + q * (BK * 128), &tmap, &full[s], i0 + q * BOX, (int)t);
#pragma unroll
        for (int q = 0; q < BN / 2 / BOX; ++q)
          tma_load_2d_pair(b + q * (BK * 128), &tmap, &full[s], j0 + (int)rank * (BN / 2) + q * BOX, (int)t);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader, one thread): chunk c into accumulator c % 2 of both
    // CTAs (rows 0-127 in the leader's TMEM, 128-255 in the peer's)
    if (lane == 0 && leader) {
      uint32_t kb = 0;
      for (int64_t c = 0; c < nchunks; ++c) {
        const uint32_t b = (uint32_t)(c & 1);
        mbar_wait(&tempty[b], ((uint32_t)(c >> 1) & 1) ^ 1);  // both folds of chunk c - 2 done
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + b * BN;
        const int64_t t1 = min(p, (c + 1) * CHUNK);
        for (int64_t t = c * CHUNK; t < t1; t += BK, ++kb) {
          const uint32_t s = kb % STAGES;
          mbar_wait(&full[s], (kb / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // 16 tokens = 16 rows of 128 B inside every 64-channel box (same offsets in both CTAs)
            const uint64_t ad = umma_desc_sw128(a_addr + kk * 2048, BK * 128, 1024);
            const uint64_t bd = umma_desc_sw128(b_addr + kk * 2048, BK * 128, 1024);
            mma_f16_pair(d_tmem, ad, bd, IDESC, (t == c * CHUNK && kk == 0) ? 0u : 1u);
          }
          mma_commit_pair_mc(&empty[s], 0x3);  // frees stage s in both CTAs when these MMAs retire
        }
        mma_commit_pair_mc(&tfull[b], 0x3);  // chunk accumulator ready for both epilogues
      }
    }
  } else {
    // ---------------- epilogue: R (128 columns of this thread's row) += chunk; store partials
    const int quarter = warp & 3;  // TMEM lanes [32 quarter, +32) are this warp's
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + half * 128;
    float R[128];
#pragma unroll
    for (int x = 0; x < 128; ++x) R[x] = 0.0f;
    for (int64_t c = 0; c < nchunks; ++c) {
      const uint32_t b = (uint32_t)(c & 1);
      mbar_wait(&tfull[b], (uint32_t)(c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        uint32_t v0[16];
        tmem_ld16(lane_base + b * BN + g * 16, v0);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 16; ++q) R[g * 16 + q] = __fadd_rn(R[g * 16 + q], __uint_as_float(v0[q]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[b]);
        else mbar_arrive_remote(&tempty[b], 0);
      }
      const int64_t c1 = c + 1;
      if (c1 == nchunks || (c1 * CHUNK) % SUPER == 0) {
        // super-chunk done: store its partial (fire-and-forget) and restart R
        const int64_t sc = c / (SUPER / CHUNK);
        float* dst = Psc + ((sc * ntiles + blockIdx.x) * (int64_t)TILE_ELEMS) + (int64_t)(half * 128) * BM + row;
#pragma unroll
        for (int x = 0; x < 128; ++x) {
          dst[(int64_t)x * BM] = R[x];
          R[x] = 0.0f;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves while the pair's MMAs or signals may target it
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem_base, 512);
}

// 2^k as a double (k within the normal range)
__device__ __forceinline__ double pow2(int k) { return __longlong_as_double((long long)(1023 + k) << 52); }

// int64 sum over the super-chunks of the partials rounded onto the grid 2^(E_i + E_j - 46)
__device__ __forceinline__ long long fixed_sum(const float* __restrict__ P, int64_t nsc, int64_t stride,
                                               int shift) {
  const double sc = pow2(shift);  // exact scaling (|shift| < 300)
  long long acc = 0;
  for (int64_t k = 0; k < nsc; ++k) acc += __double2ll_rn((double)P[k * stride] * sc);
  return acc;
}

// element index of the diagonal entry (c, c) in the tile layout
__device__ __forceinline__ int64_t diag_index(int64_t c) {
  const int64_t I = c / 256, r = (c % 256) / BM;
  const int64_t tile = 2 * (I * (I + 1) / 2 + I) + r;
  return tile * TILE_ELEMS + (c % 256) * BM + (c % BM);
}

// E_c = ceil(e / 2) + 1 for D_c = max_sc P_sc[c][c] = m 2^e (m in [0.5, 1)); E_MIN for D_c = 0
__global__ void diag_exp_kernel(const float* __restrict__ Psc, int64_t nsc, int64_t n, int ntiles,
                                int32_t* __restrict__ E) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const float* d = Psc + diag_index(c);
  float D = 0.0f;
  for (int64_t k = 0; k < nsc; ++k) D = fmaxf(D, d[k * (int64_t)ntiles * TILE_ELEMS]);
  int e = 0;
  frexpf(D, &e);
  E[c] = (D > 0.0f) ? ((e + 1) >> 1) + 1 : E_MIN;
}

// Hfix (= or +=) the exact integer sum of the partials; one thread per tile element.
__global__ void __launch_bounds__(256)
hessian_fixed_kernel(const float* __restrict__ Psc, int64_t nsc, int64_t n, int ntiles, const int32_t* __restrict__ E,
                     long long* __restrict__ Hfix, int accumulate) {
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= (int64_t)ntiles * TILE_ELEMS) return;
  int row0, col0;
  tile_of((int)(e / TILE_ELEMS), row0, col0);
  const int r = (int)(e % BM), c = (int)((e % TILE_ELEMS) / BM);
  const int64_t gi = (int64_t)row0 + r, gj = (int64_t)col0 + c;
  long long v = 0;
  if (gi < n && gj <= gi)
    v = fixed_sum(Psc + e, nsc, (int64_t)ntiles * TILE_ELEMS, GRID_SHIFT - E[gi] - E[gj]);
  Hfix[e] = accumulate ? Hfix[e] + v : v;
}

// H (full symmetric fp64; += when accumulate) from the fixed-point tiles -- or, with Psc set,
// straight from the partials (single call) -- one CTA per 32 x 32 block of a tile, through a
// shared-memory transpose so both triangles are written coalesced.  Lower entries (gj <= gi)
// only: the upper half of a diagonal tile is another summation order.
__global__ void __launch_bounds__(256)
hessian_finalize_kernel(const long long* __restrict__ Hfix, const float* __restrict__ Psc, int64_t nsc,
                        const int32_t* __restrict__ E, int64_t n, double* __restrict__ H, int accumulate) {
  __shared__ double tile[32][33];
  const int ntiles = gridDim.x / ((BM / 32) * (BN / 32));
  const int id = blockIdx.x / ((BM / 32) * (BN / 32));
  const int sub = blockIdx.x % ((BM / 32) * (BN / 32));
  int row0, col0;
  tile_of(id, row0, col0);
  const int64_t ib = (int64_t)row0 + (sub / (BN / 32)) * 32;  // first row of this block
  const int64_t jb = (int64_t)col0 + (sub % (BN / 32)) * 32;  // first column
  if (jb > ib + 31 || ib >= n || jb >= n) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t tbase = (int64_t)id * TILE_ELEMS;
  // (1) lanes along i: the integer sum of the entry, scaled onto the fp64 grid
  for (int c = ty; c < 32; c += 8) {
    const int64_t gi = ib + tx, gj = jb + c;
    double v = 0.0;
    if (gi < n && gj <= gi) {
      const int64_t e = tbase + (gj - col0) * BM + (gi - row0);
      const int shift = GRID_SHIFT - E[gi] - E[gj];
      const long long fx = Psc ? fixed_sum(Psc + e, nsc, (int64_t)ntiles * TILE_ELEMS, shift) : Hfix[e];
      v = (double)fx * pow2(-shift);
    }
    tile[c][tx] = v;
  }
  __syncthreads();
  // (2) lanes along j: the lower entries H[gi][gj] (+= the old value)
  for (int r = ty; r < 32; r += 8) {
    const int64_t gi = ib + r, gj = jb + tx;
    if (gi < n && gj <= gi) {
      double v = tile[tx][r];
      if (accumulate) v += H[gi * n + gj];
      H[gi * n + gj] = v;
      tile[tx][r] = v;
    }
  }
  __syncthreads();
  // (3) lanes along i: the mirrored upper entries H[gj][gi] (strictly above the diagonal)
  for (int c = ty; c < 32; c += 8) {
    const int64_t gi = ib + tx, gj = jb + c;
    if (gi < n && gj < gi) H[gj * n + gi] = tile[c][tx];
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

int hessian_tiles(int64_t n) {
  const int T2 = (int)((n + 255) / 256);  // 256 x 256 pair blocks per dimension
  return T2 * (T2 + 1);                   // two CTAs per lower-triangle pair block
}
int64_t hessian_superchunks(int64_t p) { return (p + SUPER - 1) / SUPER; }
size_t hessian_fixed_bytes(int64_t n) { return (size_t)hessian_tiles(n) * TILE_ELEMS * sizeof(long long); }
size_t hessian_partials_bytes(int64_t p, int64_t n) {
  return (size_t)hessian_superchunks(p) * hessian_tiles(n) * TILE_ELEMS * sizeof(float);
}

ganq_status_t check_hessian_args(const uint16_t* X, int64_t p, int64_t n) {
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
  return GANQ_OK;
}

ganq_status_t launch_hessian_partials(const uint16_t* X, int64_t p, int64_t n, float* Psc, int32_t* E,
                                      cudaStream_t st) {
  ganq_status_t s = check_hessian_args(X, p, n);
  if (s) return s;
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
  GANQ_CUDA_TRY(cudaFuncSetAttribute(hessian_syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)hessian_tiles(n));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // CTA pairs (cta_group::2 MMA)
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // GANQ_HESSIAN_CHUNK (debug / measurement only): another chain length, a power of two in [64, 32768]
  static const int64_t chunk = [] {
    const char* e = getenv("GANQ_HESSIAN_CHUNK");
    const int64_t c = e ? atoll(e) : CHUNK_DEFAULT;
    return (c >= BK && c <= SUPER && (c & (c - 1)) == 0) ? c : CHUNK_DEFAULT;
  }();
  GANQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, hessian_syrk_kernel, tmap, p, n, Psc, chunk));
  GANQ_LAUNCH_CHECK("hessian_syrk_kernel");
  diag_exp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Psc, hessian_superchunks(p), n, hessian_tiles(n), E);
  GANQ_LAUNCH_CHECK("diag_exp_kernel");
  return GANQ_OK;
}

ganq_status_t launch_hessian_fixed(const float* Psc, int64_t p, int64_t n, const int32_t* E, long long* Hfix,
                                   int accumulate, cudaStream_t st) {
  const int nt = hessian_tiles(n);
  const int64_t elems = (int64_t)nt * TILE_ELEMS;
  hessian_fixed_kernel<<<(unsigned)((elems + 255) / 256), 256, 0, st>>>(Psc, hessian_superchunks(p), n, nt, E, Hfix,
                                                                        accumulate);
  GANQ_LAUNCH_CHECK("hessian_fixed_kernel");
  return GANQ_OK;
}

ganq_status_t launch_hessian_finalize(const long long* Hfix, const float* Psc, int64_t p, const int32_t* E, int64_t n,
                                      double* H, int accumulate, cudaStream_t st) {
  const unsigned blocks = (unsigned)hessian_tiles(n) * (BM / 32) * (BN / 32);
  hessian_finalize_kernel<<<blocks, 256, 0, st>>>(Hfix, Psc, Psc ? hessian_superchunks(p) : 0, E, n, H, accumulate);
  GANQ_LAUNCH_CHECK("hessian_finalize_kernel");
  return GANQ_OK;
}

}  // namespace ganq
