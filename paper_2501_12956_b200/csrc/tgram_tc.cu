// tgram_tc.cu -- the normal matrices of the T-update (Eq. 6) on the tensor cores.
//
//   G_i = S_i H S_i^T = C_i + C_i^T + D_i,   C_i[a][b] = sum_{j>k} [q_ij=a][q_ik=b] H_jk
//
// (P:143-144 batches the T-update over rows; the sums over the one-hot S_i are m n^2 / 2
// additions per iteration, the largest term of the loop.)  For a group of R = 128 / 2^N rows
// (M = 128 pairs (i, b)) we compute
//     Dt[(i,b)][j] = sum_{k<j} [q_ik = b] * H_jk            (tensor cores, int8 x int8 -> int32)
//     C_i[a][b]   += sum_j [q_ij = a] * Dt[(i,b)][j]          (sorted segmented walk, fp64)
// H's strict lower triangle is stored once per layer as 24-bit fixed point per row j
// (scale s_j = max_{k<j}|H_jk| / (2^23 - 2^16)) split into three balanced int8 digits
// (reading R-14), so the tensor-core sums are EXACT integers: the result is deterministic and
// independent of summation order.
//
// Pipeline (one CTA per (row group, j range); SPLIT CTAs per group over balanced j ranges):
//   warp 0     TMA: the three digit tiles of H (128 j x 64 k, SWIZZLE_64B) per stage
//   warp 1     MMA issuer (+TMEM owner): 3 int32 accumulators of 128 columns, A from TMEM
//   warps 2-5  one-hot producers, one per TMEM lane quarter: lane (i,b) builds its 64 bytes
//              [q_ik == b] per stage in registers and tcgen05.st's them into a TMEM ring
//              (no shared-memory traffic for A; codes prefetched one stage ahead)
//   warps 6-9  epilogue: drain TMEM (digits -> fp32 * s_j) into a shared staging tile and
//              release the accumulators at once, then the segment sums overlap the next
//              j-tile's MMAs
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int TJ = 128;          // j per tile (UMMA N)
constexpr int TK = 64;           // k per stage (64-byte swizzle rows of int8)
constexpr int STAGES = 6;
constexpr int B_TILE = TJ * TK;                  // 8 KB digit tile of H
constexpr int STAGE_BYTES = 3 * B_TILE;          // 24 KB (the one-hot A operand lives in TMEM)
constexpr int SPLIT = 4;                         // CTAs per row group (balanced j ranges)
constexpr int THREADS = 320;                     // 10 warps
constexpr int A_COL0 = 3 * TJ;                   // TMEM: 3 accumulators, then the A ring
constexpr int A_COLS = TK / 4;                   // 16 columns of 4 int8 per stage
constexpr int NCH = TJ / 32;                     // 32-column chunks per j-tile (sorting unit)
constexpr uint32_t IDESC = umma_idesc_s8(128, TJ);
constexpr double QSCALE = 8388608.0 - 65536.0;   // 2^23 - 2^16: |h_int| bound

// SW64 K-major UMMA descriptor: 64-byte rows, 8-row atoms of 512 B (SBO), layout type 4.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

template <int NLEV>
struct TcSmem {
  static constexpr int R = 128 / NLEV;
  alignas(16) float stage[128][TJ + 1];      // drained Dt tile (fp32 values), row = (i,b)
  alignas(16) uint8_t ipos[R][TJ];           // per (row, 32-chunk): sorted position of each j
  alignas(16) float scale[TJ];               // s_j of the current j-tile (fp32)
  alignas(16) uint8_t off[R][NCH][NLEV + 1]; // segment offsets per (row, chunk, level)
  alignas(8) uint64_t full[STAGES], empty[STAGES], tfull, tempty;
  uint32_t tmem_slot;
};

__host__ __device__ inline int ktiles_of(int jt) { return (jt * TJ + TJ - 1) / TK + 1; }

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
tgram_tc_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ Q,
                const double* __restrict__ scale, int64_t m, int64_t n, int64_t P,
                const int4 jsplit, double* __restrict__ Cg, int dbg) {
  constexpr int R = 128 / NLEV;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  TcSmem<NLEV>& sm = *reinterpret_cast<TcSmem<NLEV>*>(tiles + STAGES * STAGE_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)(blockIdx.x / SPLIT) * R;
  const int NT = (int)((n + TJ - 1) / TJ);
  const int part = blockIdx.x % SPLIT;
  const int bnd[SPLIT + 1] = {0, jsplit.x, jsplit.y, jsplit.z, NT};
  const int jt_lo = bnd[part], jt_hi = bnd[part + 1];
  double* Cpart = Cg + (size_t)part * (size_t)m * NLEV * NLEV;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], 1 + 4);  // TMA bytes + one arrive per producer warp
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
        for (int kt = 0; kt < ktiles_of(jt); ++kt, ++ks) {
          const uint32_t s = ks % STAGES;
          mbar_wait(&sm.empty[s], ((ks / STAGES) & 1) ^ 1);
          uint8_t* st = tiles + s * STAGE_BYTES;
          mbar_arrive_expect_tx(&sm.full[s], 3 * B_TILE);
#pragma unroll
          for (int l = 0; l < 3; ++l)
            tma_load_2d(st + l * B_TILE, &tmap, &sm.full[s], kt * TK, (int)(l * P + jt * TJ));
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      uint32_t ks = 0;
      for (int jt = jt_lo; jt < jt_hi; ++jt) {
        mbar_wait(&sm.tempty, ((jt - jt_lo) & 1) ^ 1);
        tc_fence_after();
        for (int kt = 0; kt < ktiles_of(jt); ++kt, ++ks) {
          const uint32_t s = ks % STAGES;
          mbar_wait(&sm.full[s], (ks / STAGES) & 1);
          tc_fence_after();
          const uint32_t s_addr = smem_u32(tiles + s * STAGE_BYTES);
          const uint32_t a_tmem = tmem + A_COL0 + s * A_COLS;
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            const uint32_t b_addr = s_addr + l * B_TILE;
#pragma unroll
            for (int kk = 0; kk < TK / 32; ++kk)
              mma_i8_ts(tmem + l * TJ, a_tmem + kk * 8, umma_desc_sw64(b_addr + kk * 32), IDESC,
                        (kt > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull);
      }
    }
  } else if (warp < 6) {
    // ---------------- one-hot producers: TMEM lane (i, b) <- [q_ik == b] for the stage's 64 k
    const int pl = (warp & 3) * 32 + lane;  // == TMEM lane (this warp's quarter)
    const int i = pl / NLEV, b = pl % NLEV;
    const int64_t row = r0 + i;
    const uint32_t bb = 0x01010101u * (uint32_t)b;
    const uint8_t* qrow = Q + (row < m ? row : 0) * n;
    auto load_codes = [&](int kt, uint4 (&v)[TK / 16]) {
#pragma unroll
      for (int c = 0; c < TK / 16; ++c) {
        const int64_t k = (int64_t)kt * TK + c * 16;
        v[c] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (row < m) {
          const uint8_t* src = qrow + k;
          if (k + 16 <= n && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            v[c] = __ldg(reinterpret_cast<const uint4*>(src));
          } else {
            uint8_t* vb = reinterpret_cast<uint8_t*>(&v[c]);
#pragma unroll
            for (int q = 0; q < 16; ++q) vb[q] = (k + q < n) ? src[q] : (uint8_t)0xFF;
          }
        }
      }
    };
    // byte-wise (x == b) -> 0x01 / 0x00 for codes < 16 or 0xFF: no borrow crosses a byte
    auto onehot = [&](uint32_t x) {
      const uint32_t y = (x ^ bb) | 0x80808080u;
      return (~(y - 0x01010101u) & 0x80808080u) >> 7;
    };
    uint4 cur[TK / 16], nxt[TK / 16];
    int jt = jt_lo, kt = 0;
    if (jt < jt_hi) load_codes(kt, cur);
    uint32_t ks = 0;
    while (jt < jt_hi) {
      const uint32_t s = ks % STAGES;
      int jn = jt, kn = kt + 1;
      if (kn >= ktiles_of(jn)) { ++jn; kn = 0; }
      if (jn < jt_hi) load_codes(kn, nxt);  // prefetch the next stage's codes
      uint32_t v[16];
#pragma unroll
      for (int c = 0; c < TK / 16; ++c) {
        v[4 * c + 0] = onehot(cur[c].x);
        v[4 * c + 1] = onehot(cur[c].y);
        v[4 * c + 2] = onehot(cur[c].z);
        v[4 * c + 3] = onehot(cur[c].w);
      }
      mbar_wait(&sm.empty[s], ((ks / STAGES) & 1) ^ 1);
      tc_fence_after();
      tmem_st16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + A_COL0 + s * A_COLS, v);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.full[s]);
#pragma unroll
      for (int c = 0; c < TK / 16; ++c) cur[c] = nxt[c];
      jt = jn;
      kt = kn;
      ++ks;
    }
  } else {
    // ---------------- epilogue
    const int quarter = warp & 3;          // TMEM lane quarter of this warp
    const int et = quarter * 32 + lane;    // 0..127 == TMEM lane == (i, b)
    const int i = et / NLEV, b = et % NLEV;
    double acc[NLEV];
#pragma unroll
    for (int a = 0; a < NLEV; ++a) acc[a] = 0.0;
    for (int jt = jt_lo; jt < jt_hi; ++jt) {
      const int64_t J0 = (int64_t)jt * TJ;
      // (1) sorted order of each row's 32-column chunks (counting sort by code); overlaps MMA
      constexpr int NTASK = (R * NCH + 3) / 4;
      int codes[NTASK];
#pragma unroll
      for (int u = 0; u < NTASK; ++u) {
        const int task = quarter + 4 * u;
        const int ri = task / NCH, c = task % NCH;
        const int64_t row = r0 + ri, j = J0 + c * 32 + lane;
        codes[u] = (task < R * NCH && row < m && j < n) ? (int)__ldg(Q + row * n + j) : 0xFF;
      }
#pragma unroll
      for (int u = 0; u < NTASK; ++u) {
        const int task = quarter + 4 * u;
        if (task >= R * NCH) break;
        const int ri = task / NCH, c = task % NCH;
        const int code = codes[u];
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
        // invalid columns (j >= n, rows >= m) go after every segment
        sm.ipos[ri][c * 32 + lane] = (uint8_t)(pos >= 0 ? pos : 31);
      }
      if (et < TJ) sm.scale[et] = (J0 + et < n) ? (float)scale[J0 + et] : 0.0f;
      named_bar_sync(1, 128);
      // (2) drain: exact int32 digit sums -> fp32 (* s_j) into the staging tile, release TMEM
      mbar_wait(&sm.tfull, (jt - jt_lo) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int g = 0; g < TJ / 16; ++g) {
        uint32_t d0[16], d1[16], d2[16];
        const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + g * 16;
        tmem_ld16(tb, d0);
        tmem_ld16(tb + TJ, d1);
        tmem_ld16(tb + 2 * TJ, d2);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const float v = fmaf((float)(int)d0[t], 65536.0f,
                               fmaf((float)(int)d1[t], 256.0f, (float)(int)d2[t]));
          const int x = g * 16 + t;  // write in sorted order within its 32-column chunk
          sm.stage[et][(x & ~31) + sm.ipos[i][x]] = v * sm.scale[x];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty);  // the next j-tile's MMAs may start now
      // (3) segment sums over this thread's own (sorted) staging row: prefix sums in place,
      //     segment a of chunk c = P[off[a+1]] - P[off[a]]
#pragma unroll 1
      for (int c = 0; c < ((dbg & 1) ? 0 : NCH); ++c) {
        float* row = &sm.stage[et][c * 32];
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = row[q];
        float p = 0.0f;
        row[0] = 0.0f;
#pragma unroll
        for (int q = 0; q < 31; ++q) {
          p += v[q];
          row[q + 1] = p;  // P[q + 1]; P[32] is never needed (segments end <= 31 < 32?)
        }
        const float ptot = p + v[31];
#pragma unroll
        for (int a = 0; a < NLEV; ++a) {
          const int s0 = sm.off[i][c][a], s1 = sm.off[i][c][a + 1];
          const float hi = (s1 == 32) ? ptot : row[s1];
          const float lo = row[s0];  // s0 <= 31
          acc[a] += (s1 > s0) ? (double)(hi - lo) : 0.0;
        }
      }
      named_bar_sync(1, 128);  // perm/off/scale/stage are rewritten for the next j-tile
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
  cuuint32_t box[2] = {TK, TJ};  // 64 k (bytes) x 128 j
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)Hq, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(GANQ_ERR_CUDA, "tgram: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GANQ_ERR_CUDA;
  }
  constexpr int R = 128 / NLEV;
  const size_t smem = 1024 + STAGES * STAGE_BYTES + sizeof(TcSmem<NLEV>);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(tgram_tc_kernel<NLEV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  // split the j-tiles (work of tile jt = ktiles_of(jt)) into SPLIT ranges of equal work
  const int NT = (int)((n + TJ - 1) / TJ);
  int64_t total = 0;
  for (int jt = 0; jt < NT; ++jt) total += ktiles_of(jt);
  int bnd[SPLIT - 1];
  int64_t acc = 0;
  int jt = 0;
  for (int p = 1; p < SPLIT; ++p) {
    while (jt < NT && SPLIT * (acc + ktiles_of(jt)) <= p * total) acc += ktiles_of(jt++);
    bnd[p - 1] = jt;
  }
  const int4 jsplit = make_int4(bnd[0], bnd[1], bnd[2], 0);
  const unsigned groups = (unsigned)((m + R - 1) / R);
  static const int dbg = getenv("GANQ_TGRAM_DBG") ? atoi(getenv("GANQ_TGRAM_DBG")) : 0;
  tgram_tc_kernel<NLEV><<<SPLIT * groups, THREADS, smem, st>>>(tmap, Q, scale, m, n, P, jsplit, Cg, dbg);
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
