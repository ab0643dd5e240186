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
// computed in exact integer arithmetic on tcgen05.mma kind::i8 (reading R-15): per 64-u block
// both operands are 24-bit fixed point with their own scale (LhatT per (column, block), E per
// (row, block)), split into three balanced int8 digits; the six digit products of weight
// >= 2^16 go to three int32 TMEM accumulators (weights 2^32, 2^24, 2^16), exact in any order.  The
// reader warps scale each block's integer sums and add them in fp32 registers.  Blocks are
// issued oldest first, so the feedback of panel q-1 runs while panel q is still being decided;
// only its last 2 blocks wait for panel q's residuals.  The panel group makes the 128
// sequential decisions per panel with the in-panel feedback in fp32 FMA, and quantizes each
// finished 64-column half of residuals for the tensor cores.
//
// Warps: 0 = TMA producer, 1 = MMA issuer (+TMEM owner), 2-5 = TMEM readers (one lane
// quarter each), 6-9 = panel group (4 lanes per row).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int RB = 32;              // rows per CTA (UMMA N)
constexpr int PW = 128;             // panel width (UMMA M)
constexpr int UB = 64;              // u per feedback block (64-byte SW64 rows of int8 digits)
constexpr int STAGES = 3;
constexpr int NBUF = 4;             // TMEM accumulator sets of 3 x 32 columns (weights 2^16, 2^8, 1)
constexpr int BUF_COLS = 3 * RB;
constexpr int CS = 4;               // cluster size: row groups sharing each LhatT tile (multicast)
constexpr uint16_t CMASK = (1u << CS) - 1u;
constexpr int A_TILE = PW * UB;     // 8 KB: one digit of LhatT (128 panel columns x 64 u)
constexpr int B_TILE = RB * UB;     // 2 KB: one digit of E (32 rows x 64 u)
constexpr int STAGE_BYTES = 3 * A_TILE + 3 * B_TILE;  // 30 KB
constexpr int THREADS = 320;   // 10 warps: TMA, MMA, 4 readers, 4 panel
constexpr uint32_t IDESC = umma_idesc_s8(PW, RB);
constexpr float QSCALE = 8388608.0f - 65536.0f;  // 2^23 - 2^16: |fixed-point value| bound
// digit products (a = LhatT digit, b = E digit, weight group 2 - (a + b)); digit 0 is the top
constexpr int NPROD = 6;
__host__ __device__ constexpr int prod_a(int p) { return p == 0 ? 0 : p == 1 ? 0 : p == 2 ? 1 : p == 3 ? 0 : p == 4 ? 1 : 2; }
__host__ __device__ constexpr int prod_b(int p) { return p == 0 ? 0 : p == 1 ? 1 : p == 2 ? 0 : p == 3 ? 2 : p == 4 ? 1 : 0; }
__host__ __device__ constexpr bool prod_first(int p) { return p == 0 || p == 1 || p == 3; }

struct SsSmem {
  alignas(128) float Ld[PW][PW];         // Lhat[jb + c][jb + c2] of the current panel (TMA)
  alignas(16) float As[2][PW][RB + 1];   // drained feedback per (panel column, row), 2 buffers
  alignas(16) float es[2 * 32][RB + 1];  // residuals of the current half panel (column, row)
  alignas(16) uint8_t cs[32][RB + 4];    // codes of the current sub-panel (column, row)
  alignas(8) uint64_t full[STAGES], empty[STAGES], tfull[NBUF], tempty[NBUF];
  alignas(8) uint64_t acc_ready[2], as_free[2], ebar, ldbar;
  uint32_t tmem_slot;
};

// debug-only cycle accounting per warp role (GANQ_SSTEP_DBG & 16)
__device__ unsigned long long g_ssprof[16];
#define TP_T0(v) long long v = (dbg & 16) ? clock64() : 0
#define TP_ACC(acc, v) do { if (dbg & 16) acc += clock64() - v; } while (0)
__device__ __forceinline__ void tp_flush(int dbg, int lane, int slot, long long v) {
  if ((dbg & 16) && lane == 0) atomicAdd(&g_ssprof[slot], (unsigned long long)v);
}

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

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
sstep_tc_kernel(const __grid_constant__ CUtensorMap tmLT, const __grid_constant__ CUtensorMap tmE,
                const __grid_constant__ CUtensorMap tmLd, const float* __restrict__ tL,
                const float* __restrict__ W, const float* __restrict__ T, int64_t m, int64_t n,
                int64_t np, int64_t npq, uint8_t* __restrict__ Q, int8_t* __restrict__ Eq,
                float* __restrict__ sE, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  SsSmem& sm = *reinterpret_cast<SsSmem*>(tiles + STAGES * STAGE_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int P = (int)((n + PW - 1) / PW);  // panels; panel q covers [n - PW(q+1), n - PW q)

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmLT);
    prefetch_tmap(&tmE);
    prefetch_tmap(&tmLd);
    // empty[s] collects one (multicast) MMA commit from every CTA of the cluster
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], CS); }
    for (int b = 0; b < NBUF; ++b) { mbar_init(&sm.tfull[b], 1); mbar_init(&sm.tempty[b], 4); }
    for (int b = 0; b < 2; ++b) { mbar_init(&sm.acc_ready[b], 4); mbar_init(&sm.as_free[b], 1); }
    mbar_init(&sm.ebar, 1);
    mbar_init(&sm.ldbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_slot, 512);
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
      TP_T0(t_all);
      long long w_empty = 0, w_ebar = 0;
      uint32_t kb = 0;
      for (int q = 1; q < P; ++q) {
        const int jb = (int)(n - (int64_t)PW * (q + 1));
        const int jbs = jb + (int)(np - n);  // fp32 Lhat storage column of the panel start
        for (int qs = 0; qs < q; ++qs) {
          if (qs == q - 1) {
            TP_T0(t1);
            mbar_wait(&sm.ebar, (uint32_t)((q - 1) & 1));  // panel q-1 residuals written
            TP_ACC(w_ebar, t1);
            mbar_arrive_expect_tx(&sm.ldbar, PW * PW * 4);  // ... and its Ld no longer read
            tma_load_2d(&sm.Ld[0][0], &tmLd, &sm.ldbar, jbs, jb);
          }
          for (int k2 = 0; k2 < PW / UB; ++k2, ++kb) {
            const int u0 = (int)(npq - (int64_t)PW * (qs + 1)) + k2 * UB;  // int8 storage column
            const uint32_t s = kb % STAGES;
            TP_T0(t0);
            mbar_wait(&sm.empty[s], ((kb / STAGES) & 1) ^ 1);
            TP_ACC(w_empty, t0);
            uint8_t* st = tiles + s * STAGE_BYTES;
            mbar_arrive_expect_tx(&sm.full[s], STAGE_BYTES);
            // this CTA's quarter of the LhatT digit tiles, multicast to the whole cluster
            const int sl = (int)crank * (PW / CS);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              tma_load_3d_mc(st + d * A_TILE + sl * UB, &tmLT, &sm.full[s], u0, jb + sl, d, CMASK);
              tma_load_3d(st + 3 * A_TILE + d * B_TILE, &tmE, &sm.full[s], u0, (int)r0, d);
            }
          }
        }
      }
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, 0, 0, tot);
      tp_flush(dbg, 0, 1, w_empty);
      tp_flush(dbg, 0, 2, w_ebar);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: one accumulator set per block (exact int32 digit sums)
    if (lane == 0) {
      TP_T0(t_all);
      long long w_te = 0, w_full = 0;
      uint32_t kb = 0;
      for (int q = 1; q < P; ++q)
        for (int qs = 0; qs < q; ++qs)
          for (int k2 = 0; k2 < PW / UB; ++k2, ++kb) {
            const uint32_t s = kb % STAGES, buf = kb % NBUF;
            TP_T0(t0);
            mbar_wait(&sm.tempty[buf], ((kb / NBUF) & 1) ^ 1);
            TP_ACC(w_te, t0);
            TP_T0(t1);
            mbar_wait(&sm.full[s], (kb / STAGES) & 1);
            TP_ACC(w_full, t1);
            tc_fence_after();
            const uint32_t st = smem_u32(tiles + s * STAGE_BYTES);
            const uint32_t d = tmem + buf * BUF_COLS;
#pragma unroll
            for (int p = 0; p < NPROD; ++p) {
              const int wgt = 2 - (prod_a(p) + prod_b(p));  // 2 -> 2^16, 1 -> 2^8, 0 -> 1
              const uint32_t a = st + prod_a(p) * A_TILE, b = st + 3 * A_TILE + prod_b(p) * B_TILE;
#pragma unroll
              for (int kk = 0; kk < UB / 32; ++kk)
                mma_i8(d + (2 - wgt) * RB, umma_desc_sw64(a + kk * 32), umma_desc_sw64(b + kk * 32), IDESC,
                       (prod_first(p) && kk == 0) ? 0u : 1u);
            }
            mma_commit_mc(&sm.empty[s], CMASK);  // frees stage s in every CTA of the cluster
            mma_commit(&sm.tfull[buf]);
          }
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, 0, 3, tot);
      tp_flush(dbg, 0, 4, w_te);
      tp_flush(dbg, 0, 5, w_full);
    }
  } else if (warp < 6) {
    // ---------------- TMEM readers: lane = panel column c, 32 fp32 partials (rows)
    const int quarter = warp & 3;
    const int c = quarter * 32 + lane;
    uint32_t kb = 0;
    TP_T0(t_all);
    long long w_tf = 0, w_af = 0;
    for (int q = 0; q < P; ++q) {
      const int64_t j = n - (int64_t)PW * (q + 1) + c;  // this lane's panel column (< 0: phantom)
      float acc[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = 0.0f;
      for (int qs = 0; qs < q; ++qs) {
        for (int k2 = 0; k2 < PW / UB; ++k2, ++kb) {
          const uint32_t buf = kb % NBUF;
          const int64_t blk = (npq - (int64_t)PW * (qs + 1)) / UB + k2;  // storage block of u
          TP_T0(t0);
          mbar_wait(&sm.tfull[buf], (kb / NBUF) & 1);
          TP_ACC(w_tf, t0);
          tc_fence_after();
          // block scales: LhatT per (column, block), E per (row, block); the digit weights of the
          // three groups are 2^32, 2^24, 2^16 = 2^16 x (65536, 256, 1)
          const float tl = (j >= 0) ? tL[blk * n + j] * 65536.0f : 0.0f;
          float se[RB];
          const float4* sp4 = reinterpret_cast<const float4*>(sE + blk * ((m + RB - 1) / RB * RB) + r0);
#pragma unroll
          for (int r4 = 0; r4 < RB / 4; ++r4) {
            const float4 v = sp4[r4];  // written by this CTA's panel group: no __ldg
            se[4 * r4 + 0] = v.x * tl;
            se[4 * r4 + 1] = v.y * tl;
            se[4 * r4 + 2] = v.z * tl;
            se[4 * r4 + 3] = v.w * tl;
          }
          // (read after tfull: the E scales of the panel just decided are stored by the panel group
          // before ebar, which orders them before this block's TMA, MMA and commit)
          const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BUF_COLS;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // rows [16 hh, 16 hh + 16): three weight groups
            uint32_t c0[16], c1[16], c2[16];
            tmem_ld16(tb + 16 * hh, c0);
            tmem_ld16(tb + RB + 16 * hh, c1);
            tmem_ld16(tb + 2 * RB + 16 * hh, c2);
            tmem_ld_wait();
            if (hh == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&sm.tempty[buf]);
            }
#pragma unroll
            for (int x = 0; x < 16; ++x) {
              const float v = fmaf((float)(int)c0[x], 65536.0f, fmaf((float)(int)c1[x], 256.0f, (float)(int)c2[x]));
              acc[16 * hh + x] = fmaf(v, se[16 * hh + x], acc[16 * hh + x]);
            }
          }
        }
      }
      const int ab = q & 1;
      TP_T0(t1);
      mbar_wait(&sm.as_free[ab], ((q >> 1) & 1) ^ 1);
      TP_ACC(w_af, t1);
#pragma unroll
      for (int r = 0; r < RB; ++r) sm.As[ab][c][r] = acc[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_ready[ab]);
    }
    long long tot = 0;
    TP_ACC(tot, t_all);
    tp_flush(dbg, lane, 6, tot);
    tp_flush(dbg, lane, 7, w_tf);
    tp_flush(dbg, lane, 8, w_af);
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
    const int64_t mq = (m + RB - 1) / RB * RB;         // rows of the sE table
    float t[LPL];
#pragma unroll
    for (int x = 0; x < LPL; ++x) {
      const int lev = sub * LPL + x;
      t[x] = (live && lev < NLEV) ? T[row * NLEV + lev] : 0.0f;
    }
    const float* wrow = W + (live ? row : 0) * n;
    const uint32_t pbar = 3;                           // named barrier of the panel group
    TP_T0(t_all);
    long long w_acc = 0, w_ld = 0, c_dec = 0, c_st = 0, c_x = 0, c_bar = 0;
    for (int q = 0; q < P; ++q) {
      const int64_t jb = n - (int64_t)PW * (q + 1);
      const int ab = q & 1;
      TP_T0(t0);
      mbar_wait(&sm.acc_ready[ab], (q >> 1) & 1);
      TP_ACC(w_acc, t0);
      TP_T0(t1);
      mbar_wait(&sm.ldbar, q & 1);
      TP_ACC(w_ld, t1);
      float wn[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t j = jb + 32 * (PW / 32 - 1) + 4 * k + sub;
        wn[k] = (j >= 0) ? wrow[j] : 0.0f;
      }
#pragma unroll 1
      for (int sp = PW / 32 - 1; sp >= 0; --sp) {
        const int64_t j0 = jb + 32 * sp;     // first column of the sub-panel (may be < 0)
        float (*esp)[RB + 1] = &sm.es[32 * (sp & 1)];  // this sub-panel's half of es
        float a[8], w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a[k] = sm.As[ab][32 * sp + 4 * k + sub][rr];
          w[k] = wn[k];
        }
        TP_T0(t2);
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
            esp[cc][rr] = ec;
            sm.cs[cc][rr] = (uint8_t)bi;
          }
          const float* lrow = &sm.Ld[32 * sp + cc][32 * sp + sub];  // Lhat[j][j0 + 4 k + sub]
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (4 * k + sub < cc) a[k] = fmaf(ec, lrow[4 * k], a[k]);
        }
        TP_ACC(c_dec, t2);
        TP_T0(t3);
        named_bar_sync(pbar, 128);  // es / cs of this sub-panel complete
        TP_ACC(c_bar, t3);
        TP_T0(t4);
        // codes: lane sub writes columns [8 sub, 8 sub + 8) of its row
        if (live) {
          uint8_t cv[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) cv[x] = sm.cs[8 * sub + x][rr];
          const int64_t jj = j0 + 8 * sub;
          uint8_t* qd = Q + row * n + jj;
          if (jj >= 0 && (reinterpret_cast<uintptr_t>(qd) & 7) == 0) {
            uint2 pk;
            pk.x = cv[0] | (cv[1] << 8) | (cv[2] << 16) | ((uint32_t)cv[3] << 24);
            pk.y = cv[4] | (cv[5] << 8) | (cv[6] << 16) | ((uint32_t)cv[7] << 24);
            *reinterpret_cast<uint2*>(qd) = pk;
          } else {
#pragma unroll
            for (int x = 0; x < 8; ++x)
              if (jj + x >= 0) qd[x] = cv[x];
          }
        }
        // a finished 64-column half of a source panel: per-row scale and int8 digits of E
        // (the leftmost panel is never a source).  Lane sub quantizes columns
        // [16 sub, 16 sub + 16) of the half; storage column = j + (npq - n), a multiple of 16.
        const int64_t hs = npq - n + jb + 32 * sp;  // storage column of the half (sp even)
        if ((sp & 1) == 0 && q < P - 1 && hs >= 0) {
          float ev[16];
          float mx = 0.0f;
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            ev[x] = sm.es[16 * sub + x][rr];
            mx = fmaxf(mx, fabsf(ev[x]));
          }
          mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, 2));
          const float scale = (mx > 0.0f) ? mx / QSCALE : 0.0f;
          const float inv = (mx > 0.0f) ? QSCALE / mx : 0.0f;
          uint32_t dg[3][4];
#pragma unroll
          for (int x4 = 0; x4 < 4; ++x4) {
            uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              int h = __float2int_rn(ev[4 * x4 + y] * inv);
              const int d2 = ((h + 128) & 255) - 128;
              h = (h - d2) >> 8;
              const int d1 = ((h + 128) & 255) - 128;
              const int d0 = (h - d1) >> 8;
              w0 |= (uint32_t)(d0 & 255) << (8 * y);
              w1 |= (uint32_t)(d1 & 255) << (8 * y);
              w2 |= (uint32_t)(d2 & 255) << (8 * y);
            }
            dg[0][x4] = w0;
            dg[1][x4] = w1;
            dg[2][x4] = w2;
          }
          if (live) {
#pragma unroll
            for (int d = 0; d < 3; ++d)
              *reinterpret_cast<uint4*>(Eq + ((int64_t)d * m + row) * npq + hs + 16 * sub) =
                  make_uint4(dg[d][0], dg[d][1], dg[d][2], dg[d][3]);
            if (sub == 0) sE[(hs / UB) * mq + row] = scale;
          }
        }
        TP_ACC(c_st, t4);
        TP_T0(t5);
        // feedback of this sub-panel into the sub-panels left of it: lane sub owns target
        // columns [8 sub, 8 sub + 8) of every earlier sub-panel
#pragma unroll 1
        for (int tp = 0; tp < sp; ++tp) {
          float ac[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) ac[x] = sm.As[ab][32 * tp + 8 * sub + x][rr];
#pragma unroll 4
          for (int cc = 0; cc < 32; ++cc) {
            const float ec = esp[cc][rr];
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
        TP_ACC(c_x, t5);
        TP_T0(t6);
        named_bar_sync(pbar, 128);  // As updated, es / cs free for the next sub-panel
        TP_ACC(c_bar, t6);
      }
      fence_proxy_async_global();  // residual digit stores -> visible to the TMA (async proxy)
      named_bar_sync(pbar, 128);
      if (pl == 0) {
        mbar_arrive(&sm.ebar);
        mbar_arrive(&sm.as_free[ab]);
      }
    }
    long long tot = 0;
    TP_ACC(tot, t_all);
    tp_flush(dbg, lane, 9, tot);
    tp_flush(dbg, lane, 10, w_acc);
    tp_flush(dbg, lane, 11, w_ld);
    tp_flush(dbg, lane, 12, c_dec);
    tp_flush(dbg, lane, 13, c_st);
    tp_flush(dbg, lane, 14, c_x);
    tp_flush(dbg, lane, 15, c_bar);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Per layer: Lhat[u][j] = L_uj / L_jj for u > j (fp32, for the in-panel feedback).  Rows have
// pitch np (multiple of 4) and are stored right-aligned: column x lives at storage column
// x + (np - n), so that every TMA box start of the panel diagonal blocks is 16-byte aligned;
// storage columns [0, np - n) are zero.
__global__ void lhat_kernel(const double* __restrict__ L, int64_t n, int64_t np, float* __restrict__ Lhat) {
  const int64_t u = blockIdx.y;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < np; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = x - (np - n);
    Lhat[u * np + x] = (j >= 0 && u > j) ? (float)(L[u * n + j] / L[j * n + j]) : 0.0f;
  }
}

// Per layer: LhatT[j][u] = L_uj / L_jj (u > j) as 24-bit fixed point per (column j, 64-u block):
// tL[blk][j] = max_{u in blk} |LhatT[j][u]| / (2^23 - 2^16) and three balanced int8 digits
// LTq[d][j][u'] (digit 0 on top) at right-aligned storage columns u' = u + (npq - n), npq a
// multiple of 64 (reading R-15).  One CTA per (32 columns j, one block of 64 u).
__global__ void __launch_bounds__(256) lhat_quant_kernel(const double* __restrict__ L, int64_t n, int64_t npq,
                                                         int8_t* __restrict__ LTq, float* __restrict__ tL) {
  __shared__ double tile[64][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t blk = blockIdx.y;
  const int64_t u0 = blk * 64 - (npq - n);  // logical u of the block's first storage column
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  {
    const int64_t j = j0 + tx;
    const double dj = (j < n) ? L[j * n + j] : 1.0;
    for (int r = ty; r < 64; r += 8) {
      const int64_t u = u0 + r;
      tile[r][tx] = (j < n && u >= 0 && u < n && u > j) ? L[u * n + j] / dj : 0.0;
    }
  }
  __syncthreads();
  constexpr double QS = 8388608.0 - 65536.0;
  for (int jj = 0; jj < 4; ++jj) {
    const int jl = ty * 4 + jj;
    const int64_t j = j0 + jl;
    if (j >= n) break;
    const double x0 = tile[tx][jl], x1 = tile[tx + 32][jl];
    double mx = fmax(fabs(x0), fabs(x1));
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float sc = (mx > 0.0) ? (float)(mx / QS) : 0.0f;
    const double inv = (mx > 0.0) ? 1.0 / (double)sc : 0.0;
    if (tx == 0) tL[blk * n + j] = sc;
    const double xs[2] = {x0, x1};
    for (int h2 = 0; h2 < 2; ++h2) {
      long long h = llrint(xs[h2] * inv);
      const int d2 = (int)(((h + 128) & 255) - 128);
      h = (h - d2) / 256;
      const int d1 = (int)(((h + 128) & 255) - 128);
      const int d0 = (int)((h - d1) / 256);
      const int64_t col = blk * 64 + 32 * h2 + tx;
      LTq[(0 * n + j) * npq + col] = (int8_t)d0;
      LTq[(1 * n + j) * npq + col] = (int8_t)d1;
      LTq[(2 * n + j) * npq + col] = (int8_t)d2;
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

// [3][outer][npq] int8 digit planes, box 64 x box_outer x 1, SWIZZLE_64B (UMMA K-major SW64)
bool make_digit_map(CUtensorMap* map, const int8_t* base, int64_t npq, int64_t outer, uint32_t box_outer) {
  auto encode = encode_fn();
  if (!encode) return false;
  cuuint64_t dims[3] = {(cuuint64_t)npq, (cuuint64_t)outer, 3};
  cuuint64_t strides[2] = {(cuuint64_t)npq, (cuuint64_t)(npq * outer)};
  cuuint32_t box[3] = {(cuuint32_t)UB, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NLEV>
ganq_status_t launch_t(const float* W, const float* Lhat, const int8_t* LTq, const float* tL, const float* T,
                       int64_t m, int64_t n, int64_t np, int64_t npq, uint8_t* Q, int8_t* Eq, float* sE,
                       cudaStream_t st) {
  CUtensorMap mLT, mE, mLd;
  // out-of-range boxes (rows >= m, panel columns < 0) are zero-filled by the TMA
  if (!make_digit_map(&mLT, LTq, npq, n, PW / CS) || !make_digit_map(&mE, Eq, npq, m, RB) ||
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
  static const int dbg = getenv("GANQ_SSTEP_DBG") ? atoi(getenv("GANQ_SSTEP_DBG")) : 0;
  GANQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, sstep_tc_kernel<NLEV>, mLT, mE, mLd, tL, W, T, m, n, np, npq, Q,
                                   Eq, sE, dbg));
  GANQ_LAUNCH_CHECK("sstep_tc_kernel");
  if (dbg & 16) {
    unsigned long long h[16];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_ssprof, sizeof(h));
    const double c = (double)((groups + CS - 1) / CS * CS);
    fprintf(stderr,
            "ssprof per CTA (kcyc): tma %.1f (empty %.1f, ebar %.1f) | mma %.1f (tempty %.1f, full %.1f) | "
            "rd/warp %.1f (tfull %.1f, as_free %.1f) | panel/warp %.1f (acc_ready %.1f, ld %.1f, dec %.1f, "
            "st %.1f, cross %.1f, bar %.1f)\n",
            h[0] / c / 1e3, h[1] / c / 1e3, h[2] / c / 1e3, h[3] / c / 1e3, h[4] / c / 1e3, h[5] / c / 1e3,
            h[6] / c / 4e3, h[7] / c / 4e3, h[8] / c / 4e3, h[9] / c / 4e3, h[10] / c / 4e3, h[11] / c / 4e3,
            h[12] / c / 4e3, h[13] / c / 4e3, h[14] / c / 4e3, h[15] / c / 4e3);
    const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_ssprof, z, sizeof(z));
  }
  return GANQ_OK;
}

}  // namespace

int64_t ss_pitch(int64_t n) { return (n + 3) / 4 * 4; }
int64_t ssq_pitch(int64_t n) { return (n + 63) / 64 * 64; }

ganq_status_t launch_lhat_prep(const double* L, int64_t n, float* Lhat, int8_t* LTq, float* tL, cudaStream_t st) {
  const int64_t np = ss_pitch(n), npq = ssq_pitch(n);
  lhat_kernel<<<dim3((unsigned)((np + 255) / 256), (unsigned)n), 256, 0, st>>>(L, n, np, Lhat);
  GANQ_LAUNCH_CHECK("lhat_kernel");
  lhat_quant_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)(npq / 64)), 256, 0, st>>>(L, n, npq, LTq, tL);
  GANQ_LAUNCH_CHECK("lhat_quant_kernel");
  return GANQ_OK;
}

ganq_status_t launch_sstep_tc(const float* W, const float* Lhat, const int8_t* LTq, const float* tL,
                              const float* T, int64_t m, int64_t n, int nlev, uint8_t* Q, int8_t* Eq,
                              float* sE, cudaStream_t st) {
  const int64_t np = ss_pitch(n), npq = ssq_pitch(n);
  switch (nlev) {
    case 2: return launch_t<2>(W, Lhat, LTq, tL, T, m, n, np, npq, Q, Eq, sE, st);
    case 4: return launch_t<4>(W, Lhat, LTq, tL, T, m, n, np, npq, Q, Eq, sE, st);
    case 8: return launch_t<8>(W, Lhat, LTq, tL, T, m, n, np, npq, Q, Eq, sE, st);
    case 16: return launch_t<16>(W, Lhat, LTq, tL, T, m, n, np, npq, Q, Eq, sE, st);
    default:
      set_error(GANQ_ERR_UNSUPPORTED, "sstep: %d levels unsupported", nlev);
      return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
