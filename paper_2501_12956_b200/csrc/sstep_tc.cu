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
// computed in exact integer arithmetic on tcgen05.mma kind::i8 (reading R-15): per SOURCE PANEL
// (128 u) both operands are 24-bit fixed point with their own scale (LhatT per (column, source
// panel), E per (row, source panel)), split into three balanced int8 digits; the six digit
// products of weight >= 2^16 are exact int32 sums: one MMA per LhatT digit against the stacked
// E digits (N = 96, 64, 32), offset so that equal weights (2^32, 2^24, 2^16) accumulate in the
// same columns.  The two 64-u blocks of a source panel accumulate in one TMEM set; the reader
// warps scale each source panel's integer sums and add them in fp32 registers.  Blocks are
// issued oldest first, so the feedback of panel q-1 runs while panel q is still being decided;
// only its last 2 blocks wait for panel q's residuals.  The panel group makes the 128
// sequential decisions per panel with the in-panel feedback in fp32 FMA, and quantizes the
// finished panel's residuals for the tensor cores.
//
// Warps (roles below): TMA producer, MMA issuer (+TMEM owner), 4 TMEM readers (one lane quarter
// each), the decision warp (lane = row), 5 helpers (in-panel feedback, codes, residual digits).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <type_traits>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int RB = 32;              // rows per CTA (UMMA N)
constexpr int PW = 128;             // panel width (UMMA M)
constexpr int SB = 8;               // decision sub-panel width
constexpr int NSUB = PW / SB;
constexpr int UB = 64;              // u per feedback block (64-byte SW64 rows of int8 digits)
constexpr int STAGES = 3;
constexpr int NBUF = 4;             // TMEM accumulator sets of 3 x 32 columns (one per source panel)
constexpr int BUF_COLS = 3 * RB;
constexpr int CS = 4;               // cluster size: row groups sharing each LhatT tile (multicast)
constexpr uint16_t CMASK = (1u << CS) - 1u;
constexpr int A_TILE = PW * UB;     // 8 KB: one digit of LhatT (128 panel columns x 64 u)
constexpr int B_TILE = RB * UB;     // 2 KB: one digit of E (32 rows x 64 u)
constexpr int STAGE_BYTES = 3 * A_TILE + 3 * B_TILE;  // 30 KB
constexpr int NHELP = 5;        // in-panel helper warps
constexpr int THREADS = 32 * (7 + NHELP);  // TMA, MMA, 4 readers, helpers, decisions
// Warp roles (a warp's scheduler = its id % 4; a TMEM reader's lane quarter = its id % 4): the
// decision warp's scheduler hosts only it, the TMA warp and one reader (the light roles), the
// helpers share the other three schedulers with the remaining readers.
constexpr int TMA_WARP = 3, MMA_WARP = 1, READER0 = 4, DECIDE_WARP = 11;
__host__ __device__ constexpr int helper_index(int w) {  // helpers: warps 0, 2, 8, 9, 10
  return w == 0 ? 0 : w == 2 ? 1 : w >= 8 && w <= 10 ? w - 6 : -1;
}
constexpr int HELPER0 = 0;  // signals the panel-end barriers
constexpr int PANEL_THREADS = 32 * (1 + NHELP);
// digit a of LhatT times the E digits b = 0 .. 2 - a: N = 32 (3 - a)
__host__ __device__ constexpr uint32_t idesc_digit(int a) { return umma_idesc_s8(PW, RB * (3 - a)); }
constexpr float QSCALE = 8388608.0f - 65536.0f;  // 2^23 - 2^16: |fixed-point value| bound

struct SsSmem {
  alignas(128) float Ld[PW][PW];         // Lhat[jb + c][jb + c2] of the current panel (TMA)
  alignas(16) float As[2][PW][RB + 1];   // drained feedback per (panel column, row), 2 buffers
  alignas(16) float es[PW][RB + 1];      // residuals of the current panel (column, row)
  alignas(16) uint8_t cs[PW][RB + 4];    // codes of the current panel (column, row)
  alignas(16) float sEn[RB];             // E scales of the newest source panel (rows)
  alignas(16) float pmx[NHELP][RB];      // per helper: max |e| of the residuals it formed this panel
  alignas(16) float ws[PW][RB + 1];      // weights of the current panel (column, row)
  alignas(8) uint64_t full[STAGES], empty[STAGES], tfull[NBUF], tempty[NBUF];
  alignas(8) uint64_t acc_ready[2], as_free[2], ebar, ldbar;
  uint32_t tmem_slot;
};

// debug-only cycle accounting per warp role: compiled with -DGANQ_KPROF, enabled at run time
// by GANQ_SSTEP_DBG & 16 (tools/ss_prof.sh); absent from the default build
__device__ unsigned long long g_ssprof[20];
#ifdef GANQ_KPROF
#define TP_T0(v) long long v = (dbg & 16) ? clock64() : 0
#define TP_ACC(acc, v) do { if (dbg & 16) acc += clock64() - v; } while (0)
#else
#define TP_T0(v) constexpr long long v = 0
#define TP_ACC(acc, v) do { (void)(acc); (void)(v); } while (0)
#endif
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

// Sorted-codebook selection: with thresholds th sorted ascending, the predicates p_s = z > th_s
// are monotone, so the selected position is found by a balanced tree of selects on p (depth
// log2 NLEV, no count or index arithmetic on the dependency chain).
template <int LO, int HI, typename V, int NLEV>
__device__ __forceinline__ V tree_select(const V (&v)[NLEV], const bool (&p)[NLEV > 1 ? NLEV - 1 : 1]) {
  if constexpr (LO == HI) {
    return v[LO];
  } else {
    constexpr int MID = (LO + HI) / 2;
    const V lo = tree_select<LO, MID>(v, p);
    const V hi = tree_select<MID + 1, HI>(v, p);
    return p[MID] ? hi : lo;
  }
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
sstep_tc_kernel(const __grid_constant__ CUtensorMap tmLT, const __grid_constant__ CUtensorMap tmE,
                const __grid_constant__ CUtensorMap tmLd, const float* __restrict__ tLp,
                const float* __restrict__ W, const float* __restrict__ T, int64_t m, int64_t n,
                int64_t np, int64_t npq, uint8_t* __restrict__ Q, int8_t* __restrict__ Eq,
                float* __restrict__ sEp, int dbg) {
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
  if (warp == MMA_WARP) tmem_alloc(&sm.tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // every CTA's barriers exist before any multicast targets them
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  const uint32_t crank = cluster_ctarank();

  if (warp == TMA_WARP) {
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
          // the newest source panel: its LhatT quarters go out (multicast) before this CTA's
          // residuals exist -- they depend on L only -- so a peer's stage is not held back by
          // this CTA's decisions; only the E digit tiles wait for ebar
          const bool newest = (qs == q - 1);
          const uint32_t kb0 = kb;
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
              if (!newest) tma_load_3d(st + 3 * A_TILE + d * B_TILE, &tmE, &sm.full[s], u0, (int)r0, d);
            }
          }
          if (newest) {
            TP_T0(t1);
            mbar_wait(&sm.ebar, (uint32_t)((q - 1) & 1));  // panel q-1 residuals written
            TP_ACC(w_ebar, t1);
            mbar_arrive_expect_tx(&sm.ldbar, PW * PW * 4);  // ... and its Ld no longer read
            tma_load_2d(&sm.Ld[0][0], &tmLd, &sm.ldbar, jbs, jb);
            for (int k2 = 0; k2 < PW / UB; ++k2) {
              const int u0 = (int)(npq - (int64_t)PW * (qs + 1)) + k2 * UB;
              const uint32_t s = (kb0 + k2) % STAGES;
              uint8_t* st = tiles + s * STAGE_BYTES;
#pragma unroll
              for (int d = 0; d < 3; ++d)
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
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer: one accumulator set per source panel (exact int32 digit sums)
    if (lane == 0) {
      TP_T0(t_all);
      long long w_te = 0, w_full = 0;
      uint32_t kb = 0;
      uint32_t dr = 0;  // drains (source panels) so far
      for (int q = 1; q < P; ++q)
        for (int qs = 0; qs < q; ++qs, ++dr) {
          const uint32_t buf = dr % NBUF;
          TP_T0(t0);
          mbar_wait(&sm.tempty[buf], ((dr / NBUF) & 1) ^ 1);
          TP_ACC(w_te, t0);
          tc_fence_after();
          const uint32_t d = tmem + buf * BUF_COLS;
          for (int k2 = 0; k2 < PW / UB; ++k2, ++kb) {
            const uint32_t s = kb % STAGES;
            TP_T0(t1);
            mbar_wait(&sm.full[s], (kb / STAGES) & 1);
            TP_ACC(w_full, t1);
            tc_fence_after();
            const uint32_t st = smem_u32(tiles + s * STAGE_BYTES);
            // one MMA per LhatT digit a against the stacked E digits [b0; b1; ...; b_{2-a}]
            // (N = 32 (3 - a)) written from column 32 a, so that product (a, b) lands in column
            // range a + b: the tensor core adds equal weights (2^32, 2^24, 2^16) in exact int32,
            // and streams each A tile once per K step
#pragma unroll
            for (int kk = 0; kk < UB / 32; ++kk)
#pragma unroll
              for (int dg = 0; dg < 3; ++dg)
                mma_i8(d + dg * RB, umma_desc_sw64(st + dg * A_TILE + kk * 32),
                       umma_desc_sw64(st + 3 * A_TILE + kk * 32), idesc_digit(dg),
                       (k2 == 0 && kk == 0 && dg == 0) ? 0u : 1u);
            mma_commit_mc(&sm.empty[s], CMASK);  // frees stage s in every CTA of the cluster
          }
          mma_commit(&sm.tfull[buf]);  // the source panel's sums are complete
        }
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, 0, 3, tot);
      tp_flush(dbg, 0, 4, w_te);
      tp_flush(dbg, 0, 5, w_full);
    }
  } else if (warp >= READER0 && warp < READER0 + 4) {
    // ---------------- TMEM readers: lane = panel column c, 32 fp32 feedback values (rows)
    const int quarter = warp & 3;
    const int c = quarter * 32 + lane;
    TP_T0(t_all);
    long long w_tf = 0, w_af = 0;
    const int64_t mq = (m + RB - 1) / RB * RB;  // rows of the sEp table
    uint32_t dr = 0;
    for (int q = 0; q < P; ++q) {
      const int64_t j = n - (int64_t)PW * (q + 1) + c;  // this lane's panel column (< 0: phantom)
      float acc[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = 0.0f;
      // scales: LhatT per (column, source panel), E per (row, source panel); the digit weights of
      // the three groups are 2^32, 2^24, 2^16 = 2^16 x (65536, 256, 1).  Scales of older source
      // panels are loaded one drain ahead (the readers may run behind the MMA, so a load issued
      // right before its tfull wait would not be hidden); those of the newest source panel
      // (qs = q - 1) come from the panel group's shared copy after tfull (ordered after its stores
      // by ebar -> TMA -> MMA -> commit).
      auto load_scales = [&](int qs, float& tl_o, float (&se_o)[RB]) {
        tl_o = __ldg(tLp + (int64_t)qs * n + (j >= 0 ? j : 0));
        if (qs != q - 1) {
          const float4* sp4 = reinterpret_cast<const float4*>(sEp + (int64_t)qs * mq + r0);
#pragma unroll
          for (int r4 = 0; r4 < RB / 4; ++r4) {
            const float4 v4 = sp4[r4];
            se_o[4 * r4 + 0] = v4.x;
            se_o[4 * r4 + 1] = v4.y;
            se_o[4 * r4 + 2] = v4.z;
            se_o[4 * r4 + 3] = v4.w;
          }
        }
      };
      float tl_n = 0.0f, se_n[RB];
      if (q > 0) load_scales(0, tl_n, se_n);
      for (int qs = 0; qs < q; ++qs, ++dr) {
        const uint32_t buf = dr % NBUF;
        const float tl = tl_n;
        float se[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) se[r] = se_n[r];
        if (qs + 1 < q) load_scales(qs + 1, tl_n, se_n);
        TP_T0(t0);
        mbar_wait(&sm.tfull[buf], (dr / NBUF) & 1);
        TP_ACC(w_tf, t0);
        tc_fence_after();
        if (qs == q - 1) {
#pragma unroll
          for (int r = 0; r < RB; ++r) se[r] = sm.sEn[r];
        }
        const float tls = (j >= 0) ? tl * 65536.0f : 0.0f;
#pragma unroll
        for (int r = 0; r < RB; ++r) se[r] *= tls;
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
          // exact int32 sums -> fp32, combined by weight.  |c0| <= 128^3 = 2^21 (one digit product of
          // 128 u) converts by the add-only 1.5 * 2^23 trick (exact on [-2^22, 2^22]).  Paired fp32
          // arithmetic on two rows at a time (the same bits as scalar code).
          const float2 mg = make_float2(-12582912.0f, -12582912.0f);
          auto cv = [](uint32_t x) { return __int_as_float((int)x + 0x4B400000); };
          // (c1 and c2 combine exactly in int32: |256 c1 + c2| < 2^31; one rounding, as the fp32
          // fma(c1, 256, c2) of the separately converted sums)
#pragma unroll
          for (int x = 0; x < 16; x += 2) {
            const float2 f0 = __fadd2_rn(make_float2(cv(c0[x]), cv(c0[x + 1])), mg);
            const float2 f12 = make_float2((float)((int)c1[x] * 256 + (int)c2[x]),
                                           (float)((int)c1[x + 1] * 256 + (int)c2[x + 1]));
            const float2 v = __ffma2_rn(f0, make_float2(65536.0f, 65536.0f), f12);
            const float2 a = __ffma2_rn(v, make_float2(se[16 * hh + x], se[16 * hh + x + 1]),
                                        make_float2(acc[16 * hh + x], acc[16 * hh + x + 1]));
            acc[16 * hh + x] = a.x;
            acc[16 * hh + x + 1] = a.y;
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
    // ---------------- panel group: the decision warp (lane = row) and the helpers, which apply
    // the feedback between sub-panels (the next sub-panel's first, handed over by a named
    // barrier), store the codes and quantize finished halves of residuals for the tensor cores.
    // named barriers: the panel end, and per sub-panel ids mod 4 (the decision warp may run
    // three sub-panels ahead of the helpers, so each id has one open phase at most)
    constexpr uint32_t BAR_PANEL = 3, BAR_ES = 4, BAR_HELP = 8, BAR_X = 9;  // ES: 4 .. 7; X: 9 .. 12
    if (warp == DECIDE_WARP) {
      // ===== decision warp.  The row's codebook sorted (stable by index); th[s] separates
      // sorted positions s and s + 1: the midpoint of two distinct values (a tie goes to the
      // lower original index), or, inside a run of equal values, the next boundary above, so
      // that q = #{s : z > th_s} lands on the first member of the nearest run.  This is the
      // argmin of Eq. 22 with first-index ties, up to the rounding of the midpoints (R-10);
      // the chosen LEVEL t_q is read off the monotone predicates z > th_s by a select tree and
      // published; the helpers turn it into the code (its first index: the first member of
      // the run) and the residual, off this warp's dependency chain.
      const int64_t row = r0 + lane;
      const bool live = row < m;
      float v[NLEV];
      int ix[NLEV];
#pragma unroll
      for (int s2 = 0; s2 < NLEV; ++s2) {
        v[s2] = live ? T[row * NLEV + s2] : 0.0f;
        ix[s2] = s2;
      }
#pragma unroll
      for (int pass = 0; pass < NLEV; ++pass)
#pragma unroll
        for (int s2 = pass & 1; s2 + 1 < NLEV; s2 += 2) {
          const bool sw = v[s2] > v[s2 + 1] || (v[s2] == v[s2 + 1] && ix[s2] > ix[s2 + 1]);
          const float tv = v[s2];
          const int ti = ix[s2];
          v[s2] = sw ? v[s2 + 1] : v[s2];
          ix[s2] = sw ? ix[s2 + 1] : ix[s2];
          v[s2 + 1] = sw ? tv : v[s2 + 1];
          ix[s2 + 1] = sw ? ti : ix[s2 + 1];
        }
      int rfirst[NLEV];  // original index of the first member of each position's run
#pragma unroll
      for (int s2 = 0; s2 < NLEV; ++s2) rfirst[s2] = (s2 > 0 && v[s2] == v[s2 - 1]) ? rfirst[s2 - 1] : ix[s2];
      constexpr int NT = NLEV - 1;
      float th[NT];
      float above = __int_as_float(0x7f800000);
#pragma unroll
      for (int s2 = NT - 1; s2 >= 0; --s2) {
        if (v[s2] == v[s2 + 1]) {
          th[s2] = above;
        } else {
          const float mid = __fmul_rn(0.5f, __fadd_rn(v[s2], v[s2 + 1]));
          // z == mid is a tie: the upper run wins it iff its first index is lower (z >= mid)
          th[s2] = (ix[s2 + 1] < rfirst[s2]) ? nextafterf(mid, -__int_as_float(0x7f800000)) : mid;
          above = th[s2];
        }
      }
      named_bar_sync(BAR_PANEL, PANEL_THREADS);  // the helpers staged panel 0's weights
      TP_T0(t_all);
      long long w_acc = 0, w_ld = 0, c_dec = 0, c_bar = 0, c_ld2 = 0, c_loop = 0;
      for (int q = 0; q < P; ++q) {
        const int ab = q & 1;
        TP_T0(t0);
        mbar_wait(&sm.acc_ready[ab], (q >> 1) & 1);
        TP_ACC(w_acc, t0);
        TP_T0(t1);
        mbar_wait(&sm.ldbar, q & 1);
        TP_ACC(w_ld, t1);
        // register-carried feedback (the helpers deliver sub-panels three or more to the right):
        // a2 = into the sub-panel being decided from the two to its right, a3 = into the next one
        // from the one after it
        float a2[SB], a3[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) a2[k] = a3[k] = 0.0f;
        // one sub-panel; TL = what is known of sp at compile time (2: sp >= 2, 1: sp == 1, 0: sp == 0),
        // so that the feedback into the next two sub-panels needs no run-time branch
        auto subpanel = [&](const int sp, auto tail) {
          constexpr int TL = decltype(tail)::value;
          TP_T0(tb);
          // the helpers' feedback from sub-panels >= sp + 3 into sp (none for the first three)
          if (sp < NSUB - 3) named_bar_sync(BAR_X + (sp & 3), PANEL_THREADS);
          TP_ACC(c_bar, tb);
          TP_T0(t2);
          float a[SB], w[SB], tv[SB], lc[SB], n1[SB], n2[SB];
#pragma unroll
          for (int cc = 1; cc < SB; ++cc) lc[cc] = sm.Ld[SB * sp + cc][SB * sp + cc - 1];  // critical path
#pragma unroll
          for (int k = 0; k < SB; ++k) {
            a[k] = __fadd_rn(sm.As[ab][SB * sp + k][lane], a2[k]);
            n1[k] = a3[k];  // into sp - 1: from sp + 1 so far, from sp below
            n2[k] = 0.0f;   // into sp - 2: from sp below
            w[k] = sm.ws[SB * sp + k][lane];
          }
          // the coefficient rows of column cc (in-sub-panel part and next-sub-panel part), loaded
          // one column ahead so that their shared-memory latency is off the decision chain
          TP_ACC(c_ld2, t2);
          TP_T0(t2b);
          float4 lr[SB / 4], ln[SB / 4], lm[SB / 4];
#pragma unroll
          for (int k4 = 0; k4 < SB / 4; ++k4) {
            lr[k4] = reinterpret_cast<const float4*>(&sm.Ld[SB * sp + SB - 1][SB * sp])[k4];
            ln[k4] = (TL >= 1) ? reinterpret_cast<const float4*>(&sm.Ld[SB * sp + SB - 1][SB * (sp - 1)])[k4]
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            lm[k4] = (TL >= 2) ? reinterpret_cast<const float4*>(&sm.Ld[SB * sp + SB - 1][SB * (sp - 2)])[k4]
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int cc = SB - 1; cc >= 0; --cc) {
            float4 lrn[SB / 4], lnn[SB / 4], lmn[SB / 4];
            if (cc > 0) {
#pragma unroll
              for (int k4 = 0; k4 < SB / 4; ++k4) {
                lrn[k4] = (4 * k4 < cc - 2) ? reinterpret_cast<const float4*>(&sm.Ld[SB * sp + cc - 1][SB * sp])[k4]
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                lnn[k4] = (TL >= 1) ? reinterpret_cast<const float4*>(&sm.Ld[SB * sp + cc - 1][SB * (sp - 1)])[k4]
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                lmn[k4] = (TL >= 2) ? reinterpret_cast<const float4*>(&sm.Ld[SB * sp + cc - 1][SB * (sp - 2)])[k4]
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
            const float z = __fadd_rn(w[cc], a[cc]);
            bool pz[NT > 0 ? NT : 1];
#pragma unroll
            for (int s2 = 0; s2 < NT; ++s2) pz[s2] = z > th[s2];
            const float tq = tree_select<0, NLEV - 1>(v, pz);
            // phantom columns (j < 0, leftmost) feed only phantom columns; the helpers zero
            // their residuals before any other use
            const float ec = __fsub_rn(w[cc], tq);
            tv[cc] = tq;  // stored after the sub-panel: no shared stores between the Ld loads
            // in-sub-panel feedback into the columns left of cc (entries >= cc are already used);
            // the coefficient of column cc - 1 (the next decision) comes from a register
            if (cc > 0) a[cc - 1] = fmaf(ec, lc[cc], a[cc - 1]);
#pragma unroll
            for (int k4 = 0; k4 < SB / 4; ++k4) {
              if (4 * k4 < cc - 1) {
                const float4 l = lr[k4];
                if (4 * k4 + 0 < cc - 1) a[4 * k4 + 0] = fmaf(ec, l.x, a[4 * k4 + 0]);
                if (4 * k4 + 1 < cc - 1) a[4 * k4 + 1] = fmaf(ec, l.y, a[4 * k4 + 1]);
                if (4 * k4 + 2 < cc - 1) a[4 * k4 + 2] = fmaf(ec, l.z, a[4 * k4 + 2]);
                if (4 * k4 + 3 < cc - 1) a[4 * k4 + 3] = fmaf(ec, l.w, a[4 * k4 + 3]);
              }
            }
            // ... and into the next two sub-panels (paired FMAs)
            const float2 ee = make_float2(ec, ec);
            auto fb = [&](const float4 (&l4)[SB / 4], float (&t)[SB]) {
#pragma unroll
              for (int k4 = 0; k4 < SB / 4; ++k4) {
                const float4 l = l4[k4];
                const float2 p01 = __ffma2_rn(ee, make_float2(l.x, l.y), make_float2(t[4 * k4 + 0], t[4 * k4 + 1]));
                const float2 p23 = __ffma2_rn(ee, make_float2(l.z, l.w), make_float2(t[4 * k4 + 2], t[4 * k4 + 3]));
                t[4 * k4 + 0] = p01.x;
                t[4 * k4 + 1] = p01.y;
                t[4 * k4 + 2] = p23.x;
                t[4 * k4 + 3] = p23.y;
              }
            };
            if constexpr (TL >= 1) fb(ln, n1);
            if constexpr (TL >= 2) fb(lm, n2);
            if (cc > 0) {
#pragma unroll
              for (int k4 = 0; k4 < SB / 4; ++k4) {
                lr[k4] = lrn[k4];
                ln[k4] = lnn[k4];
                lm[k4] = lmn[k4];
              }
            }
          }
#pragma unroll
          for (int k = 0; k < SB; ++k) {
            a2[k] = n1[k];
            a3[k] = n2[k];
          }
#pragma unroll
          for (int cc = 0; cc < SB; ++cc) sm.es[SB * sp + cc][lane] = tv[cc];  // the chosen levels
          TP_ACC(c_loop, t2b);
          TP_ACC(c_dec, t2);
          __syncwarp();
          named_bar_arrive(BAR_ES + (sp & 3), PANEL_THREADS);  // the levels of sub-panel sp are in es
        };
#pragma unroll 1
        for (int sp = NSUB - 1; sp >= 2; --sp) subpanel(sp, std::integral_constant<int, 2>{});
        subpanel(1, std::integral_constant<int, 1>{});
        subpanel(0, std::integral_constant<int, 0>{});
        TP_T0(t3);
        named_bar_sync(BAR_PANEL, PANEL_THREADS);  // the helpers finished the panel
        TP_ACC(c_bar, t3);
      }
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, lane, 9, tot);
      tp_flush(dbg, lane, 10, w_acc);
      tp_flush(dbg, lane, 11, w_ld);
      tp_flush(dbg, lane, 12, c_dec);
      tp_flush(dbg, lane, 16, c_ld2);
      tp_flush(dbg, lane, 17, c_loop);
      tp_flush(dbg, lane, 15, c_bar);
    } else {
      // ===== helpers: lane = row.  After sub-panel sp is decided, its residuals are applied to
      // every column of sub-panels <= sp - 3 (4-column chunks dealt round-robin to the warps);
      // codes leave in 32-column groups, residual digits in 64-column halves.
      const int hw = helper_index(warp);
      const int rr = lane;
      const int64_t row = r0 + rr;
      const bool live = row < m;
      const float* wrow = W + (live ? row : 0) * n;
      float Tr[NLEV];  // the row's codebook (unsorted: code = index)
#pragma unroll
      for (int s2 = 0; s2 < NLEV; ++s2) Tr[s2] = live ? T[row * NLEV + s2] : 0.0f;
      // weights of panel columns [c0, c0 + SB) of the panel starting at jb -> ws (lane = row)
      // (asynchronous copies: they complete while the decisions go on, waited for at panel end)
      auto stage_w = [&](int64_t jbp, int c0) {
#pragma unroll
        for (int k = 0; k < SB; ++k) {
          const int64_t j = jbp + c0 + k;
          if (live && j >= 0)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&sm.ws[c0 + k][rr])),
                         "l"(wrow + j) : "memory");
          else
            sm.ws[c0 + k][rr] = 0.0f;
        }
      };
      for (int c0 = hw * SB; c0 < PW; c0 += NHELP * SB) stage_w(n - PW, c0);
      asm volatile("cp.async.wait_all;" ::: "memory");
      named_bar_sync(BAR_PANEL, PANEL_THREADS);
      TP_T0(t_all);
      long long c_x = 0, c_st = 0;
      float emax = 0.0f;  // max |e| over the residuals this helper formed in the current panel
      for (int q = 0; q < P; ++q) {
        const int64_t jb = n - (int64_t)PW * (q + 1);
        const int ab = q & 1;
        mbar_wait(&sm.acc_ready[ab], (q >> 1) & 1);
        mbar_wait(&sm.ldbar, q & 1);
#pragma unroll 1
        for (int sp = NSUB - 1; sp >= 0; --sp) {
          named_bar_sync(BAR_ES + (sp & 3), PANEL_THREADS);  // the decision warp finished sub-panel sp
          // codes and residuals of sub-panel sp from the chosen levels (columns dealt round-robin):
          // code = the first index s with T_s == t_q (the decision picks the first member of a
          // run of equal levels); residual e = w - t_q, zero on phantom columns (j < 0)
          for (int cc = hw; cc < SB; cc += NHELP) {
            const float tq = sm.es[SB * sp + cc][rr];
            int iq = 0;
#pragma unroll
            for (int s2 = NLEV - 1; s2 >= 0; --s2) iq = (Tr[s2] == tq) ? s2 : iq;
            sm.cs[SB * sp + cc][rr] = (uint8_t)iq;
            const float e = (jb + SB * sp + cc >= 0) ? __fsub_rn(sm.ws[SB * sp + cc][rr], tq) : 0.0f;
            sm.es[SB * sp + cc][rr] = e;
            emax = fmaxf(emax, fabsf(e));  // the panel's scale is the max over all helpers' maxima
          }
          if (sp == 0) {
            sm.pmx[hw][rr] = emax;
            emax = 0.0f;
          }
          named_bar_sync(BAR_HELP, NHELP * 32);
          TP_T0(t4);
          if (sp >= 3) {
            float e8[SB];
#pragma unroll
            for (int cc = 0; cc < SB; ++cc) e8[cc] = sm.es[SB * sp + cc][rr];
            const int nch = SB * (sp - 2) / 4;  // 4-column chunks of the columns [0, SB (sp - 2))
            // chunks in descending order: the two of sub-panel sp - 3 (needed next by the decision
            // warp) first, then the barrier arrive, then the rest (needed later; a helper handles
            // the same chunks at every step, so their order is kept)
            const int top = nch - 1 - ((nch - 1 - hw) % NHELP + NHELP) % NHELP;  // largest c4 = hw (mod NHELP)
            // NC chunks at a time (independent FMA chains interleave); paired fp32 FMAs (FFMA2: two
            // independent round-to-nearest FMAs, the same bits as scalar code)
            auto apply = [&](int c4x, auto ncc) {
              constexpr int NC = decltype(ncc)::value;
              float2 ac[NC][2];
#pragma unroll
              for (int u = 0; u < NC; ++u) {
                const int c4 = c4x - u * NHELP;
                ac[u][0] = make_float2(sm.As[ab][4 * c4][rr], sm.As[ab][4 * c4 + 1][rr]);
                ac[u][1] = make_float2(sm.As[ab][4 * c4 + 2][rr], sm.As[ab][4 * c4 + 3][rr]);
              }
#pragma unroll
              for (int cc = 0; cc < SB; ++cc) {
                const float2 ee = make_float2(e8[cc], e8[cc]);
#pragma unroll
                for (int u = 0; u < NC; ++u) {
                  const float4 l = *reinterpret_cast<const float4*>(&sm.Ld[SB * sp + cc][4 * (c4x - u * NHELP)]);
                  ac[u][0] = __ffma2_rn(ee, make_float2(l.x, l.y), ac[u][0]);
                  ac[u][1] = __ffma2_rn(ee, make_float2(l.z, l.w), ac[u][1]);
                }
              }
#pragma unroll
              for (int u = 0; u < NC; ++u) {
                const int c4 = c4x - u * NHELP;
                sm.As[ab][4 * c4][rr] = ac[u][0].x;
                sm.As[ab][4 * c4 + 1][rr] = ac[u][0].y;
                sm.As[ab][4 * c4 + 2][rr] = ac[u][1].x;
                sm.As[ab][4 * c4 + 3][rr] = ac[u][1].y;
              }
            };
            int c4 = top;
            if (c4 >= nch - 2) {  // this helper's chunk of sub-panel sp - 3 (at most one), first
              apply(c4, std::integral_constant<int, 1>{});
              c4 -= NHELP;
            }
            __syncwarp();
            named_bar_arrive(BAR_X + ((sp - 3) & 3), PANEL_THREADS);  // sub-panel sp - 3 has all its feedback
#pragma unroll 1
            for (; c4 - NHELP >= 0; c4 -= 2 * NHELP) apply(c4, std::integral_constant<int, 2>{});
            if (c4 >= 0) apply(c4, std::integral_constant<int, 1>{});
          }
          TP_ACC(c_x, t4);
          TP_T0(t5);
          // the decision warp is past sub-panel sp: stage the next panel's weights there
          if (hw == 2 && q + 1 < P) stage_w(jb - PW, SB * sp);
          const int64_t j32 = jb + SB * sp;  // (when sp % 4 == 0) first column of a 32-group
          if (hw == 4 && live && (sp & (32 / SB - 1)) == 0) {
            const int g0 = SB * sp;
            uint32_t pw[8];
#pragma unroll
            for (int x = 0; x < 8; ++x)
              pw[x] = sm.cs[g0 + 4 * x][rr] | (sm.cs[g0 + 4 * x + 1][rr] << 8) |
                      (sm.cs[g0 + 4 * x + 2][rr] << 16) | ((uint32_t)sm.cs[g0 + 4 * x + 3][rr] << 24);
            uint8_t* qd = Q + row * n + j32;
            if (j32 >= 0 && (reinterpret_cast<uintptr_t>(qd) & 15) == 0) {
              reinterpret_cast<uint4*>(qd)[0] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
              reinterpret_cast<uint4*>(qd)[1] = make_uint4(pw[4], pw[5], pw[6], pw[7]);
            } else {
#pragma unroll
              for (int x = 0; x < 32; ++x)
                if (j32 + x >= 0) qd[x] = (uint8_t)(pw[x >> 2] >> (8 * (x & 3)));
            }
          }
          // a finished panel (the leftmost panel is never a source): per-row scale and three int8
          // digits of E (reading R-15) at storage columns j + (npq - n)
          if (hw < 4 && sp == 0 && q < P - 1) {
            // the finished panel (a source of every panel left of it): the row's scale max |e| /
            // QSCALE over its 128 columns (the helpers' running maxima, published before the
            // helper barrier of sub-panel 0) and the digits; helper hw digitises the 32 columns
            // [32 hw, 32 hw + 32)
            float mx = sm.pmx[0][rr];
#pragma unroll
            for (int h2 = 1; h2 < NHELP; ++h2) mx = fmaxf(mx, sm.pmx[h2][rr]);
            const float scale = (mx > 0.0f) ? mx / QSCALE : 0.0f;
            const float inv = (mx > 0.0f) ? QSCALE / mx : 0.0f;
            const int64_t hp = npq - n + jb;  // storage column of the panel's first column
#pragma unroll 1
            for (int x16 = 2 * hw; x16 < 2 * hw + 2; ++x16) {
              if (hp + 16 * x16 < 0) continue;  // phantom columns (zero-filled by the TMA)
              uint32_t dg[3][4];
#pragma unroll
              for (int x4 = 0; x4 < 4; ++x4) {
                uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                  int h = __float2int_rn(sm.es[16 * x16 + 4 * x4 + y][rr] * inv);
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
                  *reinterpret_cast<uint4*>(Eq + ((int64_t)d * m + row) * npq + hp + 16 * x16) =
                      make_uint4(dg[d][0], dg[d][1], dg[d][2], dg[d][3]);
              }
            }
            if (hw == 0) {
              if (live) sEp[(int64_t)q * ((m + RB - 1) / RB * RB) + row] = scale;
              sm.sEn[rr] = scale;  // the newest source panel's scales, for the readers
            }
          }
          TP_ACC(c_st, t5);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");  // the next panel's weights are in ws
        fence_proxy_async_global();  // residual digit stores -> visible to the TMA (async proxy)
        named_bar_sync(BAR_PANEL, PANEL_THREADS);
        if (warp == HELPER0 && lane == 0) {
          mbar_arrive(&sm.ebar);
          mbar_arrive(&sm.as_free[ab]);
        }
      }
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, lane, 13, c_st);
      tp_flush(dbg, lane, 14, c_x);
      (void)tot;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  tc_fence_after();
  if (warp == MMA_WARP) tmem_dealloc(tmem, 512);
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

// Per layer: LhatT[j][u] = L_uj / L_jj (u > j, u in a source panel of j) as 24-bit fixed point per
// (column j, source panel qs) (reading R-15): tLp[qs][j] = max |LhatT[j][u]| / (2^23 - 2^16) over
// the panel's u, and three balanced int8 digits LTq[d][j][u'] (digit 0 on top) at right-aligned
// storage columns u' = u + (npq - n), npq a multiple of 64; source panel qs covers the storage
// columns [npq - 128 (qs + 1), npq - 128 qs).  One CTA per (32 columns j, one block of 64 u); pass 0
// writes each block's column maxima into bmax[blk][j], lhat_panelmax_kernel combines the two
// blocks of each panel into tLp, pass 1 writes the digits.
__device__ __forceinline__ int64_t panel_of_block(int64_t blk, int64_t npq) { return (npq / 64 - 1 - blk) / 2; }

__global__ void __launch_bounds__(256) lhat_quant_kernel(const double* __restrict__ L, int64_t n, int64_t npq,
                                                         int8_t* __restrict__ LTq, float* __restrict__ bmax,
                                                         const float* __restrict__ tLp, int pass) {
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
  for (int jj = 0; jj < 4; ++jj) {
    const int jl = ty * 4 + jj;
    const int64_t j = j0 + jl;
    if (j >= n) break;
    // only the source panels of column j (right of its own panel: storage u' >= npq - 128 q_j) go
    // through the tensor cores; the in-panel entries (the largest, near the diagonal) are applied
    // in fp32 and are neither scaled nor stored here
    const int64_t qj = (n - 1 - j) / 128;
    const bool src = blk * 64 >= npq - 128 * qj;
    const double x0 = src ? tile[tx][jl] : 0.0, x1 = src ? tile[tx + 32][jl] : 0.0;
    if (pass == 0) {
      double mx = fmax(fabs(x0), fabs(x1));
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (tx == 0) bmax[blk * n + j] = (float)mx;
      continue;
    }
    const float sc = tLp[panel_of_block(blk, npq) * n + j];
    const double inv = (sc > 0.0f) ? 1.0 / (double)sc : 0.0;
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

// tLp[qs][j] = the max of panel qs's two blocks (storage blocks npq/64 - 2 qs - 1, - 2) / QSCALE,
// rounded up so that every |x| / tLp <= 2^23 - 2^16 (a block index < 0 is a phantom block: 0)
__global__ void lhat_panelmax_kernel(const float* __restrict__ bmax, int64_t n, int64_t npq, float* __restrict__ tLp) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t qs = blockIdx.y;
  if (j >= n) return;
  const int64_t b1 = npq / 64 - 1 - 2 * qs, b0 = b1 - 1;
  float mx = (b1 >= 0) ? bmax[b1 * n + j] : 0.0f;
  if (b0 >= 0) mx = fmaxf(mx, bmax[b0 * n + j]);
  tLp[qs * n + j] = (mx > 0.0f) ? __fdiv_ru(mx, QSCALE) * (1.0f + 0x1p-22f) : 0.0f;
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
ganq_status_t launch_t(const float* W, const float* Lhat, const int8_t* LTq, const float* tLp, const float* T,
                       int64_t m, int64_t n, int64_t np, int64_t npq, uint8_t* Q, int8_t* Eq, float* sEp,
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
  GANQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, sstep_tc_kernel<NLEV>, mLT, mE, mLd, tLp, W, T, m, n, np, npq, Q,
                                   Eq, sEp, dbg));
  GANQ_LAUNCH_CHECK("sstep_tc_kernel");
  if (dbg & 16) {
    unsigned long long h[20];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_ssprof, sizeof(h));
    const double c = (double)((groups + CS - 1) / CS * CS);
    fprintf(stderr,
            "ssprof per CTA (kcyc): tma %.1f (empty %.1f, ebar %.1f) | mma %.1f (tempty %.1f, full %.1f) | "
            "rd/warp %.1f (tfull %.1f, as_free %.1f) | decide %.1f (acc_ready %.1f, ld %.1f, dec %.1f, "
            "bar %.1f; sub-panel loads %.1f, column loop %.1f) | helper/warp st %.1f, cross %.1f\n",
            h[0] / c / 1e3, h[1] / c / 1e3, h[2] / c / 1e3, h[3] / c / 1e3, h[4] / c / 1e3, h[5] / c / 1e3,
            h[6] / c / 4e3, h[7] / c / 4e3, h[8] / c / 4e3, h[9] / c / 1e3, h[10] / c / 1e3, h[11] / c / 1e3,
            h[12] / c / 1e3, h[15] / c / 1e3, h[16] / c / 1e3, h[17] / c / 1e3, h[13] / c / (1e3 * NHELP), h[14] / c / (1e3 * NHELP));
    const unsigned long long z[20] = {};
    cudaMemcpyToSymbol(g_ssprof, z, sizeof(z));
  }
  return GANQ_OK;
}

}  // namespace

int64_t ss_pitch(int64_t n) { return (n + 3) / 4 * 4; }
int64_t ssq_pitch(int64_t n) { return (n + 63) / 64 * 64; }

int64_t ss_panels(int64_t n) { return (n + 127) / 128; }

ganq_status_t launch_lhat_prep(const double* L, int64_t n, float* Lhat, int8_t* LTq, float* tLp, float* bmax,
                               cudaStream_t st) {
  const int64_t np = ss_pitch(n), npq = ssq_pitch(n);
  lhat_kernel<<<dim3((unsigned)((np + 255) / 256), (unsigned)n), 256, 0, st>>>(L, n, np, Lhat);
  GANQ_LAUNCH_CHECK("lhat_kernel");
  const dim3 grid((unsigned)((n + 31) / 32), (unsigned)(npq / 64));
  lhat_quant_kernel<<<grid, 256, 0, st>>>(L, n, npq, LTq, bmax, tLp, 0);
  GANQ_LAUNCH_CHECK("lhat_quant_kernel");
  lhat_panelmax_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)ss_panels(n)), 256, 0, st>>>(bmax, n, npq, tLp);
  GANQ_LAUNCH_CHECK("lhat_panelmax_kernel");
  lhat_quant_kernel<<<grid, 256, 0, st>>>(L, n, npq, LTq, bmax, tLp, 1);
  GANQ_LAUNCH_CHECK("lhat_quant_kernel");
  return GANQ_OK;
}

ganq_status_t launch_sstep_tc(const float* W, const float* Lhat, const int8_t* LTq, const float* tLp,
                              const float* T, int64_t m, int64_t n, int nlev, uint8_t* Q, int8_t* Eq,
                              float* sEp, cudaStream_t st) {
  const int64_t np = ss_pitch(n), npq = ssq_pitch(n);
  switch (nlev) {
    case 2: return launch_t<2>(W, Lhat, LTq, tLp, T, m, n, np, npq, Q, Eq, sEp, st);
    case 4: return launch_t<4>(W, Lhat, LTq, tLp, T, m, n, np, npq, Q, Eq, sEp, st);
    case 8: return launch_t<8>(W, Lhat, LTq, tLp, T, m, n, np, npq, Q, Eq, sEp, st);
    case 16: return launch_t<16>(W, Lhat, LTq, tLp, T, m, n, np, npq, Q, Eq, sEp, st);
    default:
      set_error(GANQ_ERR_UNSUPPORTED, "sstep: %d levels unsupported", nlev);
      return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
