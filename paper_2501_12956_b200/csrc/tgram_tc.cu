// tgram_tc.cu -- the normal matrices of the T-update (Eq. 6) on the tensor cores.
//
//   G_i = S_i H S_i^T = C_i + C_i^T + D_i,   C_i[a][b] = sum_{j>k} [q_ij=a][q_ik=b] H_jk
//
// (P:143-144 batches the T-update over rows; the sums over the one-hot S_i are m n^2 / 2
// additions per iteration, the largest term of the loop.)  We compute, for a group of
// R = 128 / 2^N rows (M = 128 pairs (i, b)),
//     Dt[(i,b)][j] = sum_{k<j} [q_ik = b] * H_jk            (tensor cores, int8 x int8 -> int32)
//     C_i[a][b]   += sum_j [q_ij = a] * Dt[(i,b)][j]          (sorted segmented walk, fp64)
// H's strict lower triangle is stored once per layer as 24-bit fixed point per row j
// (scale s_j = max_{k<j}|H_jk| / (2^23 - 2^16)) split into three balanced int8 digits
// (reading R-14), so the tensor-core sums are EXACT integers: the result is deterministic and
// independent of summation order.  The one-hot operand [q_ik = b] is generated in shared
// memory from the codes, in the canonical K-major 128B-swizzled UMMA layout; the digit
// tiles of H arrive by TMA.  One CTA per row group: warp 0 = TMA, warp 1 = MMA issuer
// (+TMEM owner), warps 2-3 = one-hot producers, warps 4-7 = epilogue (TMEM lane quarter each).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int TJ = 128;          // j per tile (UMMA N)
constexpr int TK = 128;          // k per stage (one 128-byte swizzle row of int8)
constexpr int MAX_STAGES = 3;
template <int NLEV> constexpr int kStages = (NLEV == 2) ? 2 : 3;  // smem budget
constexpr int TILE_BYTES = 128 * TK;             // 16 KB (one int8 operand tile)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;      // A (one-hot) + 3 digit tiles of H
constexpr int THREADS = 256;
constexpr int NPROD = 64;                        // one-hot producer threads (warps 2-3)
constexpr uint32_t IDESC = umma_idesc_s8(128, TJ);
constexpr double QSCALE = 8388608.0 - 65536.0;   // 2^23 - 2^16: |h_int| bound

template <int NLEV>
struct TcSmem {
  static constexpr int R = 128 / NLEV;
  alignas(16) float stage[128][33];          // combined Dt chunk (32 j) per (i,b) row
  alignas(16) uint8_t perm[R][TJ];           // per (row, 32-chunk): local j sorted by code
  alignas(16) float scale[TJ];               // s_j of the current j-tile (fp32)
  alignas(16) uint8_t off[R][4][NLEV + 1];   // segment offsets per (row, chunk, level)
  alignas(8) uint64_t full[MAX_STAGES], empty[MAX_STAGES], tfull, tempty;
  uint32_t tmem_slot;
};

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
tgram_tc_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ Q,
                const double* __restrict__ scale, int64_t m, int64_t n, int64_t P, int jsplit,
                double* __restrict__ Cg) {
  constexpr int R = 128 / NLEV;
  constexpr int STAGES = kStages<NLEV>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  TcSmem<NLEV>& sm = *reinterpret_cast<TcSmem<NLEV>*>(tiles + STAGES * STAGE_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)(blockIdx.x >> 1) * R;
  const int NT = (int)((n + TJ - 1) / TJ);
  // Two CTAs per row group: j-tiles [0, jsplit) and [jsplit, NT) (balanced triangle work);
  // each writes its own partial C (summed in fixed order by the solve kernel).
  const int half = blockIdx.x & 1;
  const int jt_lo = half ? jsplit : 0, jt_hi = half ? NT : jsplit;
  double* Cpart = Cg + (size_t)half * (size_t)m * NLEV * NLEV;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], 1 + NPROD);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tfull, 1);
    mbar_init(&sm.tempty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;

  if (warp == 0) {
    // ---------------- TMA: three digit tiles of H per stage
    if (lane == 0) {
      uint32_t ks = 0;
      for (int jt = jt_lo; jt < jt_hi; ++jt)
        for (int kt = 0; kt <= jt; ++kt, ++ks) {
          const uint32_t s = ks % STAGES;
          mbar_wait(&sm.empty[s], ((ks / STAGES) & 1) ^ 1);
          uint8_t* st = tiles + s * STAGE_BYTES;
          mbar_arrive_expect_tx(&sm.full[s], 3 * TILE_BYTES);
#pragma unroll
          for (int l = 0; l < 3; ++l)
            tma_load_2d(st + (1 + l) * TILE_BYTES, &tmap, &sm.full[s], kt * TK, (int)(l * P + jt * TJ));
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      uint32_t ks = 0;
      for (int jt = jt_lo; jt < jt_hi; ++jt) {
        mbar_wait(&sm.tempty, ((jt - jt_lo) & 1) ^ 1);
        tc_fence_after();
        for (int kt = 0; kt <= jt; ++kt, ++ks) {
          const uint32_t s = ks % STAGES;
          mbar_wait(&sm.full[s], (ks / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(tiles + s * STAGE_BYTES);
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            const uint32_t b_addr = a_addr + (1 + l) * TILE_BYTES;
#pragma unroll
            for (int kk = 0; kk < TK / 32; ++kk) {
              const uint64_t ad = umma_desc_sw128(a_addr + kk * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(b_addr + kk * 32, 16, 1024);
              mma_i8(tmem + l * TJ, ad, bd, IDESC, (kt > 0 || kk > 0) ? 1u : 0u);
            }
          }
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull);
      }
    }
  } else if (warp < 4) {
    // ---------------- one-hot producers: A[(i,b)][k] = [q_ik == b] (int8), K-major SW128.
    // Thread pt owns (row i, 16-column chunk c) pairs and writes the NLEV one-hot rows of
    // each; its 16 code bytes are loaded one k-tile ahead (no shared staging, no barriers).
    const int pt = threadIdx.x - 64;  // 0..63
    constexpr int PAIRS = R * (TK / 16) / NPROD;  // (i, c) pairs per thread = 16 / NLEV
    auto load_codes = [&](int kt, uint4 (&v)[PAIRS]) {
#pragma unroll
      for (int u = 0; u < PAIRS; ++u) {
        const int pr = pt + NPROD * u;
        const int i = pr / (TK / 16), c = pr % (TK / 16);
        const int64_t row = r0 + i, k = (int64_t)kt * TK + c * 16;
        v[u] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (row < m) {
          const uint8_t* src = Q + row * n + k;
          if (k + 16 <= n && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            v[u] = __ldg(reinterpret_cast<const uint4*>(src));
          } else {
            uint8_t* vb = reinterpret_cast<uint8_t*>(&v[u]);
#pragma unroll
            for (int q = 0; q < 16; ++q) vb[q] = (k + q < n) ? src[q] : (uint8_t)0xFF;
          }
        }
      }
    };
    uint4 cur[PAIRS], nxt[PAIRS];
    int jt = jt_lo, kt = 0;
    if (jt < jt_hi) load_codes(kt, cur);
    uint32_t ks = 0;
    while (jt < jt_hi) {
      const uint32_t s = ks % STAGES;
      int jn = jt, kn = kt + 1;
      if (kn > jn) { ++jn; kn = 0; }
      if (jn < jt_hi) load_codes(kn, nxt);  // prefetch the next k-tile's codes
      mbar_wait(&sm.empty[s], ((ks / STAGES) & 1) ^ 1);
      uint8_t* A = tiles + s * STAGE_BYTES;
#pragma unroll
      for (int u = 0; u < PAIRS; ++u) {
        const int pr = pt + NPROD * u;
        const int i = pr / (TK / 16), c = pr % (TK / 16);
#pragma unroll
        for (int b = 0; b < NLEV; ++b) {
          const int rr = i * NLEV + b;
          const uint32_t bb = 0x01010101u * (uint32_t)b;
          uint4 o;
          o.x = __vcmpeq4(cur[u].x, bb) & 0x01010101u;
          o.y = __vcmpeq4(cur[u].y, bb) & 0x01010101u;
          o.z = __vcmpeq4(cur[u].z, bb) & 0x01010101u;
          o.w = __vcmpeq4(cur[u].w, bb) & 0x01010101u;
          *reinterpret_cast<uint4*>(A + rr * 128 + ((c ^ (rr & 7)) << 4)) = o;
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&sm.full[s]);
#pragma unroll
      for (int u = 0; u < PAIRS; ++u) cur[u] = nxt[u];
      jt = jn;
      kt = kn;
      ++ks;
    }
  } else {
    // ---------------- epilogue: exact integer sums -> fp32 values -> sorted segmented walk
    const int et = threadIdx.x - 128;      // 0..127 == TMEM lane == (i, b)
    const int quarter = warp & 3;          // == et / 32
    const int i = et / NLEV, b = et % NLEV;
    (void)b;
    double acc[NLEV];
#pragma unroll
    for (int a = 0; a < NLEV; ++a) acc[a] = 0.0;
    for (int jt = jt_lo; jt < jt_hi; ++jt) {
      const int64_t J0 = (int64_t)jt * TJ;
      // sorted order of each row's 32-column chunks of this j-tile (counting sort by code)
      for (int task = quarter; task < R * 4; task += 4) {
        const int ri = task >> 2, c = task & 3;
        const int64_t row = r0 + ri, j = J0 + c * 32 + lane;
        const int code = (row < m && j < n) ? (int)Q[row * n + j] : 0xFF;
        const unsigned lt = (1u << lane) - 1u;
        int base = 0, pos = -1;
#pragma unroll
        for (int a = 0; a < NLEV; ++a) {
          const unsigned bal = __ballot_sync(0xffffffffu, code == a);
          if (lane == 0) sm.off[ri][c][a] = (uint8_t)base;
          if (code == a) pos = base + __popc(bal & lt);
          base += __popc(bal);
        }
        if (lane == 0) sm.off[ri][c][NLEV] = (uint8_t)base;
        if (pos >= 0) sm.perm[ri][c * 32 + pos] = (uint8_t)lane;
      }
      if (et < TJ) sm.scale[et] = (J0 + et < n) ? (float)scale[J0 + et] : 0.0f;
      named_bar_sync(1, 128);
      mbar_wait(&sm.tfull, (jt - jt_lo) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t d0[32], d1[32], d2[32];
        const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + c * 32;
        tmem_ld32(tb, d0);
        tmem_ld32(tb + TJ, d1);
        tmem_ld32(tb + 2 * TJ, d2);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          // exact int32 digit sums -> fp32 value (one rounding per step, ~2^-24 relative)
          const float v = fmaf((float)(int)d0[t], 65536.0f,
                               fmaf((float)(int)d1[t], 256.0f, (float)(int)d2[t]));
          sm.stage[et][t] = v * sm.scale[c * 32 + t];
        }
        __syncwarp();
        // only this thread's own stage row is read below: no CTA-wide barrier needed
#pragma unroll
        for (int a = 0; a < NLEV; ++a) {
          const int s0 = sm.off[i][c][a], s1 = sm.off[i][c][a + 1];
          float s = 0.0f;
          for (int q = s0; q < s1; ++q) s += sm.stage[et][sm.perm[i][c * 32 + q]];
          acc[a] += (double)s;
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty);
      named_bar_sync(1, 128);  // perm/off/scale are rewritten for the next j-tile
    }
    const int64_t row = r0 + i;
    if (row < m) {
#pragma unroll
      for (int a = 0; a < NLEV; ++a) Cpart[(row * NLEV + a) * NLEV + b] = acc[a];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Per layer: s_j and the three balanced int8 digits of round(H_jk / s_j) for k < j (else 0).
// Hq is [3][P][P] (P = n rounded up to 128), row j, k contiguous.
__global__ void __launch_bounds__(256) tq_prep_kernel(const double* __restrict__ H, int64_t n, int64_t P,
                                                      int8_t* __restrict__ Hq, double* __restrict__ scale) {
  const int64_t j = blockIdx.x;
  __shared__ double red[8];
  double mx = 0.0;
  if (j < n)
    for (int64_t k = threadIdx.x; k < j; k += blockDim.x) mx = fmax(mx, fabs(H[j * n + k]));
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < 8; ++w) mx = fmax(mx, red[w]);
  const double s = (mx > 0.0) ? mx / QSCALE : 1.0;
  if (threadIdx.x == 0) scale[j] = (j < n) ? s : 0.0;
  const double inv = 1.0 / s;
  for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
    int d0 = 0, d1 = 0, d2 = 0;
    if (j < n && k < j) {
      long long h = llrint(H[j * n + k] * inv);
      d2 = (int)(((h + 128) & 255) - 128);
      h = (h - d2) / 256;
      d1 = (int)(((h + 128) & 255) - 128);
      h = (h - d1) / 256;
      d0 = (int)h;
    }
    Hq[(0 * P + j) * P + k] = (int8_t)d0;
    Hq[(1 * P + j) * P + k] = (int8_t)d1;
    Hq[(2 * P + j) * P + k] = (int8_t)d2;
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

template <int NLEV>
ganq_status_t launch_t(const int8_t* Hq, const double* scale, const uint8_t* Q, int64_t m, int64_t n,
                       int64_t P, double* Cg, cudaStream_t st) {
  auto encode = encode_fn();
  if (!encode) {
    set_error(GANQ_ERR_CUDA, "tgram: cuTensorMapEncodeTiled unavailable");
    return GANQ_ERR_CUDA;
  }
  CUtensorMap tmap;
  cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)(3 * P)};
  cuuint64_t strides[1] = {(cuuint64_t)P};
  cuuint32_t box[2] = {TK, TJ};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)Hq, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(GANQ_ERR_CUDA, "tgram: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GANQ_ERR_CUDA;
  }
  constexpr int R = 128 / NLEV;
  const size_t smem = 1024 + kStages<NLEV> * STAGE_BYTES + sizeof(TcSmem<NLEV>);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(tgram_tc_kernel<NLEV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  // split the triangle of j-tiles (work of tile jt ~ jt + 1) into two halves of equal work
  const int NT = (int)((n + TJ - 1) / TJ);
  const int64_t total = (int64_t)NT * (NT + 1) / 2;
  int jsplit = 0;
  int64_t acc = 0;
  while (jsplit < NT && 2 * (acc + jsplit + 1) <= total) acc += ++jsplit;
  const unsigned groups = (unsigned)((m + R - 1) / R);
  tgram_tc_kernel<NLEV><<<2 * groups, THREADS, smem, st>>>(tmap, Q, scale, m, n, P, jsplit, Cg);
  GANQ_LAUNCH_CHECK("tgram_tc_kernel");
  return GANQ_OK;
}

}  // namespace

int64_t tq_pitch(int64_t n) { return (n + 127) / 128 * 128; }

ganq_status_t launch_tq_prep(const double* H, int64_t n, int8_t* Hq, double* scale, cudaStream_t st) {
  const int64_t P = tq_pitch(n);
  tq_prep_kernel<<<(unsigned)P, 256, 0, st>>>(H, n, P, Hq, scale);
  GANQ_LAUNCH_CHECK("tq_prep_kernel");
  return GANQ_OK;
}

ganq_status_t launch_tgram_tc(const int8_t* Hq, const double* scale, const uint8_t* Q, int64_t m,
                              int64_t n, int nlev, double* Cg, cudaStream_t st) {
  const int64_t P = tq_pitch(n);
  switch (nlev) {
    case 2: return launch_t<2>(Hq, scale, Q, m, n, P, Cg, st);
    case 4: return launch_t<4>(Hq, scale, Q, m, n, P, Cg, st);
    case 8: return launch_t<8>(Hq, scale, Q, m, n, P, Cg, st);
    case 16: return launch_t<16>(Hq, scale, Q, m, n, P, Cg, st);
    default:
      set_error(GANQ_ERR_UNSUPPORTED, "tgram: %d levels unsupported", nlev);
      return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
