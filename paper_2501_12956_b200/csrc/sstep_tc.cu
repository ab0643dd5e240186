// sstep_tc.cu -- the S-update (Eqs. 15-22; Algorithm 1 inner loop) with the
// blocked error feedback on the 5th-gen tensor cores.
//
// For row i, column j (n-1 down to 0):  z_ij = W_ij + a_ij,  a_ij = sum_{u>j} E_iu Lhat_uj,
// Lhat_uj = L_uj / L_jj (reading R-10);  Q_ij = argmin_s |z_ij - T_is| (first index on ties);
// E_ij = W_ij - T_{i,Q_ij} (the paper's residual r_j).
//
// One CTA owns 32 rows and sweeps 128-column panels right to left.  The feedback of panel q
// from every column right of it is a dense contraction
//     A_q[c][r] = sum_u LhatT[jb_q + c][u] * E[r][u]          (M = 128 panel columns,
//                                                            N = 32 rows, K = u)
// computed with tcgen05.mma kind::tf32 in split precision (x3: lo*hi + hi*lo + hi*hi, reading
// R-10/R-15), operands by TMA in the canonical K-major 128B-swizzled layout.  Tensor-core
// fp32 accumulation is not round-to-nearest, so every 32-u block gets its own TMEM buffer
// (<= 12 MMAs per chain) and reader warps add the block partials in fp32 registers.  Blocks
// are issued oldest first, so the feedback of panel q-1 runs while panel q is still being
// decided; only its last 4 blocks wait for panel q's residuals.  One warp (lane = row) makes
// the 128 sequential decisions per panel with the in-panel feedback in fp32 FMA.
//
// Warps: 0 = TMA producer, 1 = MMA issuer (+TMEM owner), 2-5 = TMEM readers (one lane
// quarter each), 6 = panel (decisions).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int RB = 32;              // rows per CTA (UMMA N)
constexpr int PW = 128;             // panel width (UMMA M)
constexpr int UB = 32;              // u per block (128 B of fp32: one swizzle row)
constexpr int STAGES = 3;
constexpr int NBUF = 8;             // TMEM accumulator buffers (32 columns each)
constexpr int A_BYTES = PW * UB * 4;   // 16 KB
constexpr int B_BYTES = RB * UB * 4;   // 4 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int THREADS = 224;
constexpr uint32_t IDESC = umma_idesc(/*tf32*/ 2, 0, 0, PW, RB);

struct SsSmem {
  alignas(128) float Ld[PW][PW];         // Lhat[jb + c][jb + c2] of the current panel (TMA)
  alignas(16) float As[2][PW][RB + 1];   // drained feedback per (panel column, row), 2 buffers
  alignas(16) float es[32][RB + 1];      // residuals of the current sub-panel (column, row)
  alignas(8) uint64_t full[STAGES], empty[STAGES], tfull[NBUF], tempty[NBUF];
  alignas(8) uint64_t acc_ready[2], as_free[2], ebar, ldbar;
  uint32_t tmem_slot;
};

template <int NLEV>
__device__ __forceinline__ void argmin_tree(float z, const float (&t)[NLEV], int& q, float& tq) {
  float d[NLEV];
  int idx[NLEV];
  float tv[NLEV];
#pragma unroll
  for (int s = 0; s < NLEV; ++s) {
    d[s] = fabsf(__fsub_rn(z, t[s]));
    idx[s] = s;
    tv[s] = t[s];
  }
#pragma unroll
  for (int w = 1; w < NLEV; w <<= 1) {
#pragma unroll
    for (int s = 0; s + w < NLEV; s += 2 * w) {
      const bool right = d[s + w] < d[s];
      d[s] = right ? d[s + w] : d[s];
      idx[s] = right ? idx[s + w] : idx[s];
      tv[s] = right ? tv[s + w] : tv[s];
    }
  }
  q = idx[0];
  tq = tv[0];
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
sstep_tc_kernel(const __grid_constant__ CUtensorMap tmLhi, const __grid_constant__ CUtensorMap tmLlo,
                const __grid_constant__ CUtensorMap tmEhi, const __grid_constant__ CUtensorMap tmElo,
                const __grid_constant__ CUtensorMap tmLd, const float* __restrict__ W,
                const float* __restrict__ T,
                int64_t m, int64_t n, int64_t np, uint8_t* __restrict__ Q, float* __restrict__ Ehi,
                float* __restrict__ Elo) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  SsSmem& sm = *reinterpret_cast<SsSmem*>(tiles + STAGES * STAGE_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int P = (int)((n + PW - 1) / PW);  // panels; panel q covers [n - PW(q+1), n - PW q)

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmLhi);
    prefetch_tmap(&tmLlo);
    prefetch_tmap(&tmEhi);
    prefetch_tmap(&tmElo);
    prefetch_tmap(&tmLd);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], 1); }
    for (int b = 0; b < NBUF; ++b) { mbar_init(&sm.tfull[b], 1); mbar_init(&sm.tempty[b], 4); }
    for (int b = 0; b < 2; ++b) { mbar_init(&sm.acc_ready[b], 4); mbar_init(&sm.as_free[b], 1); }
    mbar_init(&sm.ebar, 1);
    mbar_init(&sm.ldbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_slot, NBUF * RB);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: blocks of target q = 1..P-1, source panels oldest first
    if (lane == 0) {
      // diagonal block of panel 0 (the panel warp waits on ldbar, one phase per panel)
      mbar_arrive_expect_tx(&sm.ldbar, PW * PW * 4);
      tma_load_2d(&sm.Ld[0][0], &tmLd, &sm.ldbar, (int)(np - PW), (int)(n - PW));
      uint32_t kb = 0;
      for (int q = 1; q < P; ++q) {
        const int jb = (int)(n - (int64_t)PW * (q + 1));
        const int jbs = jb + (int)(np - n);  // storage column of the panel start (multiple of 4)
        for (int qs = 0; qs < q; ++qs) {
          if (qs == q - 1) {
            mbar_wait(&sm.ebar, (uint32_t)((q - 1) & 1));  // panel q-1 residuals written
            mbar_arrive_expect_tx(&sm.ldbar, PW * PW * 4);  // ... and its Ld no longer read
            tma_load_2d(&sm.Ld[0][0], &tmLd, &sm.ldbar, jbs, jb);
          }
          for (int k4 = 0; k4 < PW / UB; ++k4, ++kb) {
            const int u0 = (int)(np - (int64_t)PW * (qs + 1)) + k4 * UB;  // storage column
            const uint32_t s = kb % STAGES;
            mbar_wait(&sm.empty[s], ((kb / STAGES) & 1) ^ 1);
            uint8_t* st = tiles + s * STAGE_BYTES;
            mbar_arrive_expect_tx(&sm.full[s], STAGE_BYTES);
            tma_load_2d(st, &tmLhi, &sm.full[s], u0, jb);
            tma_load_2d(st + A_BYTES, &tmLlo, &sm.full[s], u0, jb);
            tma_load_2d(st + 2 * A_BYTES, &tmEhi, &sm.full[s], u0, (int)r0);
            tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tmElo, &sm.full[s], u0, (int)r0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: one TMEM buffer per block (short accumulation chains)
    if (lane == 0) {
      uint32_t kb = 0;
      for (int q = 1; q < P; ++q)
        for (int qs = 0; qs < q; ++qs)
          for (int k4 = 0; k4 < PW / UB; ++k4, ++kb) {
            const uint32_t s = kb % STAGES, buf = kb % NBUF;
            mbar_wait(&sm.tempty[buf], ((kb / NBUF) & 1) ^ 1);
            mbar_wait(&sm.full[s], (kb / STAGES) & 1);
            tc_fence_after();
            const uint32_t st = smem_u32(tiles + s * STAGE_BYTES);
            const uint32_t a_hi = st, a_lo = st + A_BYTES, b_hi = st + 2 * A_BYTES,
                           b_lo = st + 2 * A_BYTES + B_BYTES;
            const uint32_t d = tmem + buf * RB;
            // small terms first (lo*hi, hi*lo), then hi*hi: each chain is <= 12 MMAs
#pragma unroll
            for (int pass = 0; pass < 3; ++pass) {
              const uint32_t a = (pass == 0) ? a_lo : a_hi;
              const uint32_t b = (pass == 1) ? b_lo : b_hi;
#pragma unroll
              for (int kk = 0; kk < UB / 8; ++kk) {
                const uint64_t ad = umma_desc_sw128(a + kk * 32, 16, 1024);
                const uint64_t bd = umma_desc_sw128(b + kk * 32, 16, 1024);
                mma_tf32(d, ad, bd, IDESC, (pass > 0 || kk > 0) ? 1u : 0u);
              }
            }
            mma_commit(&sm.empty[s]);
            mma_commit(&sm.tfull[buf]);
          }
    }
  } else if (warp < 6) {
    // ---------------- TMEM readers: lane = panel column c, 32 fp32 partials (rows)
    const int quarter = warp & 3;
    const int c = quarter * 32 + lane;
    uint32_t kb = 0;
    for (int q = 0; q < P; ++q) {
      float acc[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = 0.0f;
      for (int blk = 0; blk < 4 * q; ++blk, ++kb) {
        const uint32_t buf = kb % NBUF;
        mbar_wait(&sm.tfull[buf], (kb / NBUF) & 1);
        tc_fence_after();
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + buf * RB, v);
        tmem_ld_wait();
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] += __uint_as_float(v[r]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[buf]);
      }
      const int ab = q & 1;
      mbar_wait(&sm.as_free[ab], ((q >> 1) & 1) ^ 1);
#pragma unroll
      for (int r = 0; r < RB; ++r) sm.As[ab][c][r] = acc[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_ready[ab]);
    }
  } else {
    // ---------------- panel warp: lane = row, sequential decisions
    const int64_t row = r0 + lane;
    const bool live = row < m;
    float t[NLEV];
#pragma unroll
    for (int s = 0; s < NLEV; ++s) t[s] = live ? T[row * NLEV + s] : 0.0f;
    const float* wrow = W + (live ? row : 0) * n;
    for (int q = 0; q < P; ++q) {
      const int64_t jb = n - (int64_t)PW * (q + 1);
      const int ab = q & 1;
      mbar_wait(&sm.acc_ready[ab], (q >> 1) & 1);
      mbar_wait(&sm.ldbar, q & 1);
#pragma unroll 1
      for (int sp = PW / 32 - 1; sp >= 0; --sp) {
        const int64_t j0 = jb + 32 * sp;     // first column of the sub-panel (may be < 0)
        float a[32], w[32];
        uint8_t code[32];
#pragma unroll
        for (int x = 0; x < 32; ++x) {
          a[x] = sm.As[ab][32 * sp + x][lane];
          w[x] = (j0 + x >= 0) ? wrow[j0 + x] : 0.0f;
        }
#pragma unroll
        for (int cc = 31; cc >= 0; --cc) {
          const float z = __fadd_rn(w[cc], a[cc]);
          int qv;
          float tq;
          argmin_tree<NLEV>(z, t, qv, tq);
          const bool real = j0 + cc >= 0;
          const float ec = real ? __fsub_rn(w[cc], tq) : 0.0f;
          sm.es[cc][lane] = ec;
          code[cc] = (uint8_t)qv;
          const float* lrow = &sm.Ld[32 * sp + cc][32 * sp];  // Lhat[j][j0 + c2] (0 if OOB)
#pragma unroll
          for (int c2 = 0; c2 < cc; ++c2) a[c2] = fmaf(ec, lrow[c2], a[c2]);
        }
        if (live) {
#pragma unroll
          for (int x = 0; x < 32; ++x) {
            const int64_t j = j0 + x;
            if (j >= 0) {
              Q[row * n + j] = code[x];
              const float ex = sm.es[x][lane];
              const float hi = tf32_rna(ex);
              Ehi[row * np + (np - n) + j] = hi;
              Elo[row * np + (np - n) + j] = __fsub_rn(ex, hi);
            }
          }
        }
        // feedback of this sub-panel into the sub-panels left of it (same panel)
#pragma unroll 1
        for (int tp = 0; tp < sp; ++tp) {
          float ac[32];
#pragma unroll
          for (int x = 0; x < 32; ++x) ac[x] = sm.As[ab][32 * tp + x][lane];
#pragma unroll 2
          for (int cc = 0; cc < 32; ++cc) {
            const float ec = sm.es[cc][lane];
            const float4* lrow = reinterpret_cast<const float4*>(&sm.Ld[32 * sp + cc][32 * tp]);
#pragma unroll
            for (int x4 = 0; x4 < 8; ++x4) {
              const float4 l = lrow[x4];
              ac[4 * x4 + 0] = fmaf(ec, l.x, ac[4 * x4 + 0]);
              ac[4 * x4 + 1] = fmaf(ec, l.y, ac[4 * x4 + 1]);
              ac[4 * x4 + 2] = fmaf(ec, l.z, ac[4 * x4 + 2]);
              ac[4 * x4 + 3] = fmaf(ec, l.w, ac[4 * x4 + 3]);
            }
          }
#pragma unroll
          for (int x = 0; x < 32; ++x) sm.As[ab][32 * tp + x][lane] = ac[x];
        }
        __syncwarp();
      }
      fence_proxy_async_global();  // residual stores -> visible to the TMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sm.ebar);
        mbar_arrive(&sm.as_free[ab]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, NBUF * RB);
}

// Per layer: LhatT_hi/lo[j][u] = split(L_uj / L_jj) for u > j (tf32 hi + fp32 remainder) and
// Lhat[u][j] (fp32, for the in-panel feedback).  Rows have pitch np (multiple of 4) and are
// stored right-aligned: column x lives at storage column x + (np - n), so that every TMA box
// start (n - 128 q + 32 k) is 16-byte aligned; storage columns [0, np - n) are zero.
__global__ void lhat_split_kernel(const double* __restrict__ L, int64_t n, int64_t np,
                                  float* __restrict__ Lhat, float* __restrict__ LThi,
                                  float* __restrict__ LTlo) {
  __shared__ float tile[32][33];
  __shared__ float tlo[32][33];
  const int64_t u0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t u = u0 + r, j = j0 + tx;
    float hi = 0.0f, lo = 0.0f, v = 0.0f;
    if (u < n && j < n && u > j) {
      const double x = L[u * n + j] / L[j * n + j];
      v = (float)x;
      uint32_t hb;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
      hi = __uint_as_float(hb);
      lo = (float)(x - (double)hi);
    }
    if (u < n && j < n) Lhat[u * np + (np - n) + j] = v;
    if (u < n && j < np - n) Lhat[u * np + j] = 0.0f;
    tile[r][tx] = hi;
    tlo[r][tx] = lo;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t j = j0 + r, u = u0 + tx;  // LT[j][u] = Lhat[u][j]
    if (j < n && u < n) {
      LThi[j * np + (np - n) + u] = tile[tx][r];
      LTlo[j * np + (np - n) + u] = tlo[tx][r];
    }
    if (j < n && u < np - n) {
      LThi[j * np + u] = 0.0f;
      LTlo[j * np + u] = 0.0f;
    }
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

bool make_map(CUtensorMap* map, const float* base, int64_t inner, int64_t outer, int64_t pitch_elems,
              uint32_t box_inner, uint32_t box_outer, bool swizzle = true) {
  auto encode = encode_fn();
  if (!encode) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)pitch_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE,
                swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NLEV>
ganq_status_t launch_t(const float* W, const float* Lhat, const float* LThi, const float* LTlo,
                       const float* T, int64_t m, int64_t n, int64_t np, uint8_t* Q, float* Ehi,
                       float* Elo, cudaStream_t st) {
  CUtensorMap mLhi, mLlo, mEhi, mElo, mLd;
  // inner extent = the padded pitch np (>= 4 elements: TMA needs >= 16 bytes per row); the
  // padding columns are zero (LhatT, Lhat) or never inside a box (E: u-blocks end below n)
  if (!make_map(&mLhi, LThi, np, n, np, UB, PW) || !make_map(&mLlo, LTlo, np, n, np, UB, PW) ||
      !make_map(&mEhi, Ehi, np, m, np, UB, RB) || !make_map(&mElo, Elo, np, m, np, UB, RB) ||
      !make_map(&mLd, Lhat, np, n, np, PW, PW, /*swizzle*/ false)) {
    set_error(GANQ_ERR_CUDA, "sstep: tensor map encoding failed");
    return GANQ_ERR_CUDA;
  }
  const size_t smem = 1024 + STAGES * STAGE_BYTES + sizeof(SsSmem);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(sstep_tc_kernel<NLEV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  sstep_tc_kernel<NLEV><<<(unsigned)((m + RB - 1) / RB), THREADS, smem, st>>>(
      mLhi, mLlo, mEhi, mElo, mLd, W, T, m, n, np, Q, Ehi, Elo);
  GANQ_LAUNCH_CHECK("sstep_tc_kernel");
  return GANQ_OK;
}

}  // namespace

int64_t ss_pitch(int64_t n) { return (n + 3) / 4 * 4; }

ganq_status_t launch_lhat_split(const double* L, int64_t n, float* Lhat, float* LThi, float* LTlo,
                                cudaStream_t st) {
  const int64_t np = ss_pitch(n);
  dim3 grid((unsigned)((np + 31) / 32), (unsigned)((n + 31) / 32));
  lhat_split_kernel<<<grid, dim3(32, 8), 0, st>>>(L, n, np, Lhat, LThi, LTlo);
  GANQ_LAUNCH_CHECK("lhat_split_kernel");
  return GANQ_OK;
}

ganq_status_t launch_sstep_tc(const float* W, const float* Lhat, const float* LThi, const float* LTlo,
                              const float* T, int64_t m, int64_t n, int nlev, uint8_t* Q, float* Ehi,
                              float* Elo, cudaStream_t st) {
  const int64_t np = ss_pitch(n);
  switch (nlev) {
    case 2: return launch_t<2>(W, Lhat, LThi, LTlo, T, m, n, np, Q, Ehi, Elo, st);
    case 4: return launch_t<4>(W, Lhat, LThi, LTlo, T, m, n, np, Q, Ehi, Elo, st);
    case 8: return launch_t<8>(W, Lhat, LThi, LTlo, T, m, n, np, Q, Ehi, Elo, st);
    case 16: return launch_t<16>(W, Lhat, LThi, LTlo, T, m, n, np, Q, Ehi, Elo, st);
    default:
      set_error(GANQ_ERR_UNSUPPORTED, "sstep: %d levels unsupported", nlev);
      return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
