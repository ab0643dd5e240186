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
// quarter each), 6-9 = panel group (4 lanes per row).
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
constexpr int CS = 4;               // cluster size: row groups sharing each LhatT tile (multicast)
constexpr uint16_t CMASK = (1u << CS) - 1u;
constexpr int A_BYTES = PW * UB * 4;   // 16 KB
constexpr int B_BYTES = RB * UB * 4;   // 4 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int THREADS = 320;   // 10 warps: TMA, MMA, 4 readers, 4 panel
constexpr uint32_t IDESC = umma_idesc(/*tf32*/ 2, 0, 0, PW, RB);

struct SsSmem {
  alignas(128) float Ld[PW][PW];         // Lhat[jb + c][jb + c2] of the current panel (TMA)
  alignas(16) float As[2][PW][RB + 1];   // drained feedback per (panel column, row), 2 buffers
  alignas(16) float es[32][RB + 1];      // residuals of the current sub-panel (column, row)
  alignas(16) uint8_t cs[32][RB + 4];    // codes of the current sub-panel (column, row)
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
    // empty[s] collects one (multicast) MMA commit from every CTA of the cluster
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], CS); }
    for (int b = 0; b < NBUF; ++b) { mbar_init(&sm.tfull[b], 1); mbar_init(&sm.tempty[b], 4); }
    for (int b = 0; b < 2; ++b) { mbar_init(&sm.acc_ready[b], 4); mbar_init(&sm.as_free[b], 1); }
    mbar_init(&sm.ebar, 1);
    mbar_init(&sm.ldbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_slot, NBUF * RB);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // every CTA's barriers exist before any multicast targets them
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  const uint32_t crank = cluster_ctarank();

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
            // this CTA's quarter of the LhatT hi/lo tiles, multicast to the whole cluster
            const int sl = (int)crank * (PW / CS);
            tma_load_2d_mc(st + sl * 128, &tmLhi, &sm.full[s], u0, jb + sl, CMASK);
            tma_load_2d_mc(st + A_BYTES + sl * 128, &tmLlo, &sm.full[s], u0, jb + sl, CMASK);
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
            mma_commit_mc(&sm.empty[s], CMASK);  // frees stage s in every CTA of the cluster
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
    // ---------------- panel group (warps 6-9): 4 lanes per row, sequential decisions.
    // Lane (r, sub) holds levels [4 sub, 4 sub + 4) of row r's codebook and the accumulators
    // of the sub-panel columns c = 4 k + sub.  Per column: the owner lane's z and w are
    // broadcast, each lane takes the argmin over its 4 levels, two shuffle rounds combine the
    // candidates (distance, then index: the first index wins ties exactly as in a sequential
    // strict '<' scan), and every lane forms e = w - t_q and updates its own accumulators.
    constexpr int LPL = NLEV / 4 > 0 ? NLEV / 4 : 1;   // levels per lane
    const int pl = threadIdx.x - 192;                  // 0..127
    const int rr = pl >> 2, sub = pl & 3;              // row within CTA, quarter
    const int64_t row = r0 + rr;
    const bool live = row < m;
    const unsigned gmask = 0xffffffffu;
    const int gbase = lane & ~3;                       // first lane of this row's group
    float t[LPL];
#pragma unroll
    for (int x = 0; x < LPL; ++x) {
      const int lev = sub * LPL + x;
      t[x] = (live && lev < NLEV) ? T[row * NLEV + lev] : 0.0f;
    }
    const float* wrow = W + (live ? row : 0) * n;
    const int64_t off = np - n;                        // right-aligned storage offset
    const uint32_t pbar = 3;                           // named barrier of the panel group
    for (int q = 0; q < P; ++q) {
      const int64_t jb = n - (int64_t)PW * (q + 1);
      const int ab = q & 1;
      mbar_wait(&sm.acc_ready[ab], (q >> 1) & 1);
      mbar_wait(&sm.ldbar, q & 1);
      float wn[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t j = jb + 32 * (PW / 32 - 1) + 4 * k + sub;
        wn[k] = (j >= 0) ? wrow[j] : 0.0f;
      }
#pragma unroll 1
      for (int sp = PW / 32 - 1; sp >= 0; --sp) {
        const int64_t j0 = jb + 32 * sp;     // first column of the sub-panel (may be < 0)
        float a[8], w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a[k] = sm.As[ab][32 * sp + 4 * k + sub][rr];
          w[k] = wn[k];
        }
        if (sp > 0) {  // prefetch the next sub-panel's weights
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int64_t j = j0 - 32 + 4 * k + sub;
            wn[k] = (j >= 0) ? wrow[j] : 0.0f;
          }
        }
#pragma unroll
        for (int cc = 31; cc >= 0; --cc) {
          const int own = cc & 3, kc = cc >> 2;
          const float zl = __fadd_rn(w[kc], a[kc]);                       // valid on the owner
          const float z = __shfl_sync(gmask, zl, gbase | own);
          const float wc = __shfl_sync(gmask, w[kc], gbase | own);
          // local argmin over this lane's levels (first index on ties)
          float bd = fabsf(__fsub_rn(z, t[0]));
          int bi = sub * LPL;
          float bt = t[0];
#pragma unroll
          for (int x = 1; x < LPL; ++x) {
            const float d = fabsf(__fsub_rn(z, t[x]));
            const bool better = d < bd;
            bd = better ? d : bd;
            bi = better ? sub * LPL + x : bi;
            bt = better ? t[x] : bt;
          }
          if (NLEV < 4 && sub * LPL >= NLEV) bd = __int_as_float(0x7f800000);  // no levels here
#pragma unroll
          for (int o = 1; o < 4; o <<= 1) {
            const float od = __shfl_xor_sync(gmask, bd, o);
            const int oi = __shfl_xor_sync(gmask, bi, o);
            const float ot = __shfl_xor_sync(gmask, bt, o);
            const bool take = (od < bd) || (od == bd && oi < bi);
            bd = take ? od : bd;
            bi = take ? oi : bi;
            bt = take ? ot : bt;
          }
          const bool real = j0 + cc >= 0;
          const float ec = real ? __fsub_rn(wc, bt) : 0.0f;
          if (sub == own) {
            sm.es[cc][rr] = ec;
            sm.cs[cc][rr] = (uint8_t)bi;
          }
          const float* lrow = &sm.Ld[32 * sp + cc][32 * sp + sub];  // Lhat[j][j0 + 4 k + sub]
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (4 * k + sub < cc) a[k] = fmaf(ec, lrow[4 * k], a[k]);
        }
        named_bar_sync(pbar, 128);  // es / cs of this sub-panel complete
        // stores: lane sub writes columns [8 sub, 8 sub + 8) of its row
        if (live) {
          float ev[8];
          uint8_t cv[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            ev[x] = sm.es[8 * sub + x][rr];
            cv[x] = sm.cs[8 * sub + x][rr];
          }
          const int64_t jj = j0 + 8 * sub;
          if (jj >= 0) {
            float* eh = Ehi + row * np + off + jj;
            float* el = Elo + row * np + off + jj;
            float hi[8], lo[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              hi[x] = tf32_rna(ev[x]);
              lo[x] = __fsub_rn(ev[x], hi[x]);
            }
            // storage column off + jj is a multiple of 4 (right-aligned pitch): 16-byte stores
            reinterpret_cast<float4*>(eh)[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
            reinterpret_cast<float4*>(eh)[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
            reinterpret_cast<float4*>(el)[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
            reinterpret_cast<float4*>(el)[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
            uint8_t* qd = Q + row * n + jj;
            if ((reinterpret_cast<uintptr_t>(qd) & 7) == 0) {
              uint2 pk;
              pk.x = cv[0] | (cv[1] << 8) | (cv[2] << 16) | ((uint32_t)cv[3] << 24);
              pk.y = cv[4] | (cv[5] << 8) | (cv[6] << 16) | ((uint32_t)cv[7] << 24);
              *reinterpret_cast<uint2*>(qd) = pk;
            } else {
#pragma unroll
              for (int x = 0; x < 8; ++x) qd[x] = cv[x];
            }
          } else {
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              const int64_t j = jj + x;
              if (j >= 0) {
                const float hi = tf32_rna(ev[x]);
                Ehi[row * np + off + j] = hi;
                Elo[row * np + off + j] = __fsub_rn(ev[x], hi);
                Q[row * n + j] = cv[x];
              }
            }
          }
        }
        // feedback of this sub-panel into the sub-panels left of it: lane sub owns target
        // columns [8 sub, 8 sub + 8) of every earlier sub-panel
#pragma unroll 1
        for (int tp = 0; tp < sp; ++tp) {
          float ac[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) ac[x] = sm.As[ab][32 * tp + 8 * sub + x][rr];
#pragma unroll 4
          for (int cc = 0; cc < 32; ++cc) {
            const float ec = sm.es[cc][rr];
            const float4* lrow = reinterpret_cast<const float4*>(&sm.Ld[32 * sp + cc][32 * tp + 8 * sub]);
            const float4 l0 = lrow[0], l1 = lrow[1];
            ac[0] = fmaf(ec, l0.x, ac[0]);
            ac[1] = fmaf(ec, l0.y, ac[1]);
            ac[2] = fmaf(ec, l0.z, ac[2]);
            ac[3] = fmaf(ec, l0.w, ac[3]);
            ac[4] = fmaf(ec, l1.x, ac[4]);
            ac[5] = fmaf(ec, l1.y, ac[5]);
            ac[6] = fmaf(ec, l1.z, ac[6]);
            ac[7] = fmaf(ec, l1.w, ac[7]);
          }
#pragma unroll
          for (int x = 0; x < 8; ++x) sm.As[ab][32 * tp + 8 * sub + x][rr] = ac[x];
        }
        named_bar_sync(pbar, 128);  // As updated, es / cs free for the next sub-panel
      }
      fence_proxy_async_global();  // residual stores -> visible to the TMA (async proxy)
      named_bar_sync(pbar, 128);
      if (pl == 0) {
        mbar_arrive(&sm.ebar);
        mbar_arrive(&sm.as_free[ab]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
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
  if (!make_map(&mLhi, LThi, np, n, np, UB, PW / CS) || !make_map(&mLlo, LTlo, np, n, np, UB, PW / CS) ||
      !make_map(&mEhi, Ehi, np, m, np, UB, RB) || !make_map(&mElo, Elo, np, m, np, UB, RB) ||
      !make_map(&mLd, Lhat, np, n, np, PW, PW, /*swizzle*/ false)) {
    set_error(GANQ_ERR_CUDA, "sstep: tensor map encoding failed");
    return GANQ_ERR_CUDA;
  }
  const size_t smem = 1024 + STAGES * STAGE_BYTES + sizeof(SsSmem);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(sstep_tc_kernel<NLEV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  const unsigned groups = (unsigned)((m + RB - 1) / RB);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((groups + CS - 1) / CS * CS);  // whole clusters; extra CTAs own no rows
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GANQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, sstep_tc_kernel<NLEV>, mLhi, mLlo, mEhi, mElo, mLd, W, T, m, n,
                                   np, Q, Ehi, Elo));
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
