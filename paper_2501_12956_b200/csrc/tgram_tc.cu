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
// Pipeline (one CTA per (row group, j range); tgram_splits() CTAs per group over balanced j ranges; the
// two CTAs of a cluster hold consecutive row groups and share every H tile by multicast):
//   warp 0     TMA: the three digit tiles of H (128 j x 128 k, SWIZZLE_128B) per stage
//   warp 1     MMA issuer (+TMEM owner): 3 int32 accumulators of 128 columns, A from TMEM; one
//              elected lane issues a stage's 12 MMAs and its commit in one asm block
//   warps 2-5  one-hot producers, one per TMEM lane quarter: lane (i,b) builds its 128 bytes
//              [q_ik == b] per stage in registers and tcgen05.st's them into a TMEM ring.  The
//              NLEV lanes of a row each load 1/NLEV of the row's codes, PD stages ahead, and
//              exchange them by shuffles (a global load per stage and lane was the producers'
//              stall: its latency exceeded one stage)
//   warps 6-13 epilogue, two warps per lane quarter (one per column half): drain TMEM
//              (digits -> fp32 * s_j) into a shared staging tile and release the accumulators
//              at once, then the segment sums overlap the next j-tile's MMAs
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int TJ = 128;          // j per tile (UMMA N)
constexpr int TK = 128;          // k per stage (128-byte swizzle rows of int8)
constexpr int B_TILE = TJ * TK;                  // 16 KB digit tile of H
constexpr int STAGE_BYTES = 3 * B_TILE;          // 48 KB (the one-hot A operand lives in TMEM)
constexpr int SPLIT = 4;                         // max CTAs per row group (balanced j ranges)
constexpr int CS = 2;                            // cluster: CS row groups share every H tile
constexpr uint16_t CMASK = (1u << CS) - 1;
constexpr int SLICE = TJ / CS;                   // j rows of each digit tile one CTA loads
constexpr int THREADS = 448;                     // 14 warps
constexpr int A_COL0 = 3 * TJ;                   // TMEM: 3 accumulators, then the A ring
constexpr int A_COLS = TK / 4;                   // 32 columns of 4 int8 per stage
constexpr int NCH = TJ / 32;                     // 32-column chunks per j-tile (sorting unit)
constexpr uint32_t IDESC = umma_idesc_u8s8(128, TJ);  // A = one-hot bytes 0 / 1 (u8)
constexpr double QSCALE = 8388608.0 - 65536.0;   // 2^23 - 2^16: |h_int| bound
constexpr int SROW = TJ + 4;                     // staging row pitch (16-byte aligned rows)
// pipeline depth: 3 stages; 2 at N = 1, whose sort tables (64 rows) fill the rest of shared memory
__host__ __device__ constexpr int stages_of(int nlev) { return nlev <= 2 ? 2 : 3; }
static_assert(A_COL0 + 3 * A_COLS <= 512, "accumulators and the A ring fit TMEM");

// debug-only cycle accounting per warp role: compiled with -DGANQ_KPROF, enabled at run time
// by GANQ_TGRAM_DBG & 16 (tools/tg_prof.sh); absent from the default build
__device__ unsigned long long g_tgprof[16];
#ifdef GANQ_KPROF
#define TP_T0(v) long long v = (dbg & 16) ? clock64() : 0
#define TP_ACC(acc, v) do { if (dbg & 16) acc += clock64() - v; } while (0)
#else
#define TP_T0(v) constexpr long long v = 0
#define TP_ACC(acc, v) do { (void)(acc); (void)(v); } while (0)
#endif
__device__ __forceinline__ void tp_flush(int dbg, int lane, int slot, long long v) {
  if ((dbg & 16) && lane == 0) atomicAdd(&g_tgprof[slot], (unsigned long long)v);
}

template <int NLEV>
struct TcSmem {
  static constexpr int R = 128 / NLEV;
  static constexpr int STAGES = stages_of(NLEV);
  static constexpr int NLEVP = NLEV < 4 ? 4 : NLEV;
  alignas(16) float stage[128][SROW];         // drained Dt tile (fp32 values), row = (i,b)
  // double-buffered per j-tile (the sort of tile t + 1 runs while other warps walk tile t)
  alignas(16) uint8_t perm[2][R][TJ];         // per (row, 32-chunk): the column at each sorted slot
  alignas(16) float scale[2][TJ];             // s_j of the j-tile (fp32)
  alignas(16) uint8_t oend[2][R][NCH][NLEVP]; // end of each level's segment per (row, chunk)
  alignas(8) uint64_t full[STAGES], empty[STAGES], tfull, tempty;
  uint32_t tmem_slot;
};

__host__ __device__ inline int ktiles_of(int jt) { return (jt * TJ + TJ - 1) / TK + 1; }
static_assert(TJ % TK == 0, "producers step ktiles_of by TJ / TK");

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
tgram_tc_kernel(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ Q,
                const double* __restrict__ scale, int64_t m, int64_t n, int64_t P,
                const int4 jsplit, int nsplit, int gp, double* __restrict__ Cg, int dbg) {
  constexpr int R = 128 / NLEV;
  constexpr int STAGES = stages_of(NLEV);
  constexpr int NB = NLEV == 2 ? 1 : NLEV == 4 ? 2 : NLEV == 8 ? 3 : 4;  // code bits
  static_assert((1 << NB) == NLEV, "levels are a power of two");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  TcSmem<NLEV>& sm = *reinterpret_cast<TcSmem<NLEV>*>(tiles + STAGES * STAGE_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // blockIdx.x = part * gp + group (gp = groups rounded up to whole clusters): the CS CTAs of a
  // cluster hold consecutive row groups of the same j range and share each stage's H tiles
  const int64_t r0 = (int64_t)(blockIdx.x % gp) * R;
  const int NT = (int)((n + TJ - 1) / TJ);
  const int part = blockIdx.x / gp;
  const bool small_sums = n <= 32768;  // every int32 digit sum fits the add-only conversion
  static_assert(SPLIT == 4, "j ranges come from jsplit.x .. z");
  const int jt_lo = part == 0 ? 0 : part == 1 ? jsplit.x : part == 2 ? jsplit.y : jsplit.z;
  const int jt_hi = part + 1 == nsplit ? NT : part == 0 ? jsplit.x : part == 1 ? jsplit.y : jsplit.z;
  double* Cpart = Cg + (size_t)part * (size_t)m * NLEV * NLEV;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], 1 + 4);  // TMA bytes (all CS slices) + one arrive per producer warp
      mbar_init(&sm.empty[s], CS);    // one (multicast) MMA commit from every CTA of the cluster
    }
    mbar_init(&sm.tfull, 1);
    mbar_init(&sm.tempty, 8);
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
    // ---------------- TMA: three digit tiles of H per stage
    if (lane == 0) {
      TP_T0(t_all);
      long long w_empty = 0;
      uint32_t ks = 0;
      for (int jt = jt_lo; jt < jt_hi; ++jt)
        for (int kt = 0; kt < ktiles_of(jt); ++kt, ++ks) {
          const uint32_t s = ks % STAGES;
          TP_T0(t0);
          mbar_wait(&sm.empty[s], ((ks / STAGES) & 1) ^ 1);
          TP_ACC(w_empty, t0);
          uint8_t* st = tiles + s * STAGE_BYTES;
          mbar_arrive_expect_tx(&sm.full[s], 3 * B_TILE);
          // this CTA's slice of j rows of each digit tile, multicast to the whole cluster
#pragma unroll
          for (int l = 0; l < 3; ++l)
            tma_load_2d_mc(st + l * B_TILE + crank * SLICE * TK, &tmap, &sm.full[s], kt * TK,
                           (int)(l * P + jt * TJ + crank * SLICE), CMASK);
        }
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, 0, 0, tot);
      tp_flush(dbg, 0, 1, w_empty);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (the whole warp waits; one elected lane issues each stage)
    TP_T0(t_all);
    long long w_full = 0, w_tempty = 0;
    uint32_t s = 0, ph = 0;
    const uint64_t desc0 = umma_desc_sw128(smem_u32(tiles), 16, 1024);
    for (int jt = jt_lo; jt < jt_hi; ++jt) {
      TP_T0(t1);
      mbar_wait(&sm.tempty, ((jt - jt_lo) & 1) ^ 1);
      TP_ACC(w_tempty, t1);
      tc_fence_after();
      const int nk = ktiles_of(jt);
      for (int kt = 0; kt < nk; ++kt) {
        TP_T0(t0);
        mbar_wait(&sm.full[s], ph);
        TP_ACC(w_full, t0);
        tc_fence_after();
        __syncwarp();
        // the commit frees stage s in every CTA of the cluster
        if (!(dbg & 8))
          mma_i8_ts_stage12_mc(tmem, tmem + A_COL0 + s * A_COLS, desc0 + (uint64_t)(s * (STAGE_BYTES >> 4)),
                               IDESC, kt == 0 ? 1u : 0u, &sm.empty[s], CMASK);
        else if (lane == 0)
          mma_commit_mc(&sm.empty[s], CMASK);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      __syncwarp();
      if (lane == 0) mma_commit(&sm.tfull);
    }
    long long tot = 0;
    TP_ACC(tot, t_all);
    tp_flush(dbg, lane, 2, tot);
    tp_flush(dbg, lane, 3, w_full);
    tp_flush(dbg, lane, 4, w_tempty);
  } else if (warp < 6) {
    // ---------------- one-hot producers: TMEM lane (i, b) <- [q_ik == b] for the stage's 128 k
    // (one warp per lane quarter; kept branch-light: a lone warp per scheduler hides no latency)
    const int pl = (warp & 3) * 32 + lane;  // == TMEM lane (this warp's quarter)
    const int i = pl / NLEV, b = pl % NLEV;
    const int64_t row = r0 + i;
    const uint32_t bb = 0x01010101u * (uint32_t)b;
    const uint8_t* qrow = Q + (row < m ? row : 0) * n;
    // this lane's share of its row's 128 codes per stage: WPL words at byte offset 4 WPL b
    constexpr int WPL = 32 / NLEV;
    constexpr int PD = NLEV >= 8 ? 4 : 2;  // stages whose codes are in flight
    const int row_lane0 = lane & ~(NLEV - 1);  // the row's first lane in this warp
    const bool vec = row < m && (n & 15) == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0;
    auto load_share = [&](int kt, uint32_t (&w)[WPL]) {
      const int64_t k0 = (int64_t)kt * TK + 4 * WPL * b;
      if (vec && k0 + 4 * WPL <= n) {
        if constexpr (WPL == 1) {
          w[0] = __ldg(reinterpret_cast<const uint32_t*>(qrow + k0));
        } else if constexpr (WPL == 2) {
          const uint2 x = __ldg(reinterpret_cast<const uint2*>(qrow + k0));
          w[0] = x.x;
          w[1] = x.y;
        } else {
#pragma unroll
          for (int c = 0; c < WPL / 4; ++c) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(qrow + k0) + c);
            w[4 * c] = x.x;
            w[4 * c + 1] = x.y;
            w[4 * c + 2] = x.z;
            w[4 * c + 3] = x.w;
          }
        }
      } else {
#pragma unroll
        for (int x = 0; x < WPL; ++x) {
          uint32_t v = 0;
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            const int64_t k = k0 + 4 * x + y;
            v |= (uint32_t)((row < m && k < n) ? qrow[k] : (uint8_t)0xFF) << (8 * y);
          }
          w[x] = v;
        }
      }
    };
    // byte-wise (x == b) -> 0x80 / 0x00 for codes < 16 or 0xFF (no borrow crosses a byte):
    // y = (x ^ b) | 0x80 per byte; its low 7 bits are zero iff x == b, so ~(y - 1) keeps bit 7
    // exactly then; shifted down to 0x01 (a unit one-hot keeps every digit sum below 2^22 for
    // n <= 32768, the range of the epilogue's add-only int -> float conversion)
    auto onehot = [&](uint32_t x) {
      const uint32_t y = (x ^ bb) | 0x80808080u;
      return ((0x01010100u - y) & 0x80808080u) >> 7;  // == (~(y - 0x01010101) & 0x80808080) >> 7
    };
    // two cursors over the (j-tile, k-tile) stages: `use` (stage being produced) and `ld` (the
    // stage whose codes are loaded next, PD ahead)
    int jt = jt_lo, kt = 0, nk = ktiles_of(jt_lo);
    int ljt = jt_lo, lkt = 0, lnk = nk;
    auto load_next = [&](uint32_t (&w)[WPL]) {
      if (ljt >= jt_hi) return;
      if (!(dbg & 66)) load_share(lkt, w);  // dbg & 64: timing probe without code loads
      if (++lkt >= lnk) { ++ljt; lkt = 0; lnk += TJ / TK; }
    };
    uint32_t s = 0, ph = 0;
    TP_T0(t_all);
    long long w_empty = 0, w_st = 0;
    // one stage from the codes in cur; cur is then refilled with the codes PD stages ahead
    auto stage = [&](uint32_t (&cur)[WPL]) -> bool {
      if (jt >= jt_hi) return false;
      uint32_t v[TK / 4];
#pragma unroll
      for (int x = 0; x < TK / 4; ++x)
        v[x] = onehot(__shfl_sync(0xffffffffu, cur[x % WPL], row_lane0 + x / WPL));
      load_next(cur);
      TP_T0(t0);
      mbar_wait(&sm.empty[s], ph ^ 1);
      TP_ACC(w_empty, t0);
      tc_fence_after();
      TP_T0(t2);
      if (!(dbg & 2)) {
        const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + A_COL0 + s * A_COLS;
#pragma unroll
        for (int h16 = 0; h16 < TK / 64; ++h16) {
          uint32_t w16[16];
#pragma unroll
          for (int x = 0; x < 16; ++x) w16[x] = v[16 * h16 + x];
          tmem_st16(ta + 16 * h16, w16);
        }
        tmem_st_wait();
      }
      TP_ACC(w_st, t2);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.full[s]);
      if (++kt >= nk) { ++jt; kt = 0; nk += TJ / TK; }
      if (++s == STAGES) { s = 0; ph ^= 1; }
      return true;
    };
    uint32_t cq[PD][WPL];
#pragma unroll
    for (int d = 0; d < PD; ++d) load_next(cq[d]);
    if constexpr (PD == 4) {
      while (stage(cq[0]) && stage(cq[1]) && stage(cq[2]) && stage(cq[3])) {
      }
    } else {
      while (stage(cq[0]) && stage(cq[1])) {
      }
    }
    {
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, lane, 5, tot);
      tp_flush(dbg, lane, 6, w_empty);
      tp_flush(dbg, lane, 7, w_st);
    }
  } else {
    // ---------------- epilogue: two warps per TMEM lane quarter, each owning half the columns
    const int quarter = warp & 3;          // TMEM lane quarter of this warp
    const int h = (warp - 6) >> 2;         // column half: chunks [2h, 2h + 2) of the j-tile
    const int e = warp - 6;                // 0..7
    const int et = quarter * 32 + lane;    // 0..127 == TMEM lane == (i, b)
    const int i = et / NLEV, b = et % NLEV;
    constexpr int EPI_THREADS = 256;
    // segment sums collect in fp32 over FLUSH j-tiles (8 chunk segments), then in fp64: the
    // fp64 pipe (F2F.F64 + DADD per segment) throttled the walk
    constexpr int FLUSH = 4;
    double acc[NLEV];
    float acf[NLEV];
#pragma unroll
    for (int a = 0; a < NLEV; ++a) {
      acc[a] = 0.0;
      acf[a] = 0.0f;
    }
    TP_T0(t_all);
    long long e_sort = 0, e_wait = 0, e_drain = 0, e_walk = 0, e_bar = 0;  // e_bar: unused
    // (1) codes of a j-tile: task u of this warp = (row ri, 32-column chunk c); prefetched one
    //     tile ahead (NTASK <= 8) so that their global-load latency overlaps the walk
    constexpr int NTASK = (R * NCH + 7) / 8;
    constexpr bool PREFETCH = NTASK <= 8;
    constexpr int NCODE = PREFETCH ? NTASK : 1;
    auto load_codes = [&](int jt, int u) -> int {
      const int task = e + 8 * u;
      const int ri = task / NCH, c = task % NCH;
      const int64_t row = r0 + ri, j = (int64_t)jt * TJ + c * 32 + lane;
      return (task < R * NCH && row < m && j < n) ? (int)__ldg(Q + row * n + j) : 0xFF;
    };
    int cn[NCODE];
    if constexpr (PREFETCH) {
#pragma unroll
      for (int u = 0; u < NTASK; ++u) cn[u] = (jt_lo < jt_hi) ? load_codes(jt_lo, u) : 0xFF;
    }
    for (int jt = jt_lo; jt < jt_hi; ++jt) {
      const int64_t J0 = (int64_t)jt * TJ;
      const int bf = (jt - jt_lo) & 1;
      TP_T0(ta);
      // counting sort of each (row, chunk) by code; overlaps the MMAs of this tile
      int cur[NCODE];
      if constexpr (PREFETCH) {
#pragma unroll
        for (int u = 0; u < NTASK; ++u) {
          cur[u] = cn[u];
          if (jt + 1 < jt_hi) cn[u] = load_codes(jt + 1, u);
        }
      }
#pragma unroll
      for (int u = 0; u < NTASK; ++u) {
        const int task = e + 8 * u;
        if (task >= R * NCH) break;
        const int ri = task / NCH, c = task % NCH;
        int code;
        if constexpr (PREFETCH) code = cur[u];
        else code = load_codes(jt, u);
        // radix ranks from one ballot per code bit: less(x) = #valid lanes with code < x, by
        // comparing the bits from the top (eq = the lanes whose higher bits equal x's so far)
        const unsigned vm = __ballot_sync(0xffffffffu, code < NLEV);
        unsigned bits[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t) bits[t] = __ballot_sync(0xffffffffu, (code >> t) & 1);
        auto less = [&](int x, unsigned& eq) {
          eq = vm;
          int cnt = 0;
#pragma unroll
          for (int t = NB - 1; t >= 0; --t) {
            if ((x >> t) & 1) {
              cnt += __popc(eq & ~bits[t]);
              eq &= bits[t];
            } else {
              eq &= ~bits[t];
            }
          }
          return cnt;
        };
        unsigned eqc;
        const int lc = less(code < NLEV ? code : 0, eqc);
        // stable position (equal codes keep column order); invalid columns (j >= n, rows >= m)
        // go after every segment
        // (slots past the valid count are never part of a segment: left unwritten)
        if (code < NLEV) sm.perm[bf][ri][c * 32 + lc + __popc(eqc & ((1u << lane) - 1u))] = (uint8_t)lane;
        if (lane < NLEV) {  // lane a: the end of level a's segment = #valid codes <= a
          unsigned e2;
          sm.oend[bf][ri][c][lane] = (uint8_t)(lane + 1 < NLEV ? less(lane + 1, e2) : __popc(vm));
        }
      }
      if (h == 0) sm.scale[bf][et] = (J0 + et < n) ? (float)scale[J0 + et] : 0.0f;
      named_bar_sync(1, EPI_THREADS);  // every warp's sort of this tile is visible
      TP_ACC(e_sort, ta);
      TP_T0(tb0);
      // (2) drain: exact int32 digit sums -> fp32 (* s_j) into the staging tile, release TMEM
      mbar_wait(&sm.tfull, (jt - jt_lo) & 1);
      TP_ACC(e_wait, tb0);
      TP_T0(tc0);
      tc_fence_after();
      // 8 columns at a time (3 x 8 accumulator words in registers)
      constexpr int DW = 8;
#pragma unroll 1
      for (int g = h * (TJ / 2 / DW); g < ((dbg & 4) ? 0 : (h + 1) * (TJ / 2 / DW)); ++g) {
        uint32_t d0[DW], d1[DW], d2[DW];
        const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + g * DW;
        tmem_ld8(tb, d0);
        tmem_ld8(tb + TJ, d1);
        tmem_ld8(tb + 2 * TJ, d2);
        // the scales of these columns; the values go to the staging row in column order (vector
        // stores: the walk reads them in sorted order)
        const float4 sa = reinterpret_cast<const float4*>(&sm.scale[bf][g * DW])[0];
        const float4 sb = reinterpret_cast<const float4*>(&sm.scale[bf][g * DW])[1];
        const float sc[DW] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
        float vv[DW];
        tmem_ld_wait();
        if (small_sums) {
          // |digit sum| <= 128 (n - 1) < 2^22: exact conversion by adding to 1.5 * 2^23 in the
          // integer domain and subtracting it in fp32 (full-rate IADD + FADD instead of I2F)
          // (paired fp32 arithmetic on two columns at a time: the same bits as scalar code)
          // the low two digits combine exactly in int32 (|256 S1 + S2| < 2^28); its one rounding to
          // fp32 (the converter, round to nearest) equals the fp32 fma(S1, 256, S2) of the
          // separately converted digits
          const float2 mg = make_float2(-12582912.0f, -12582912.0f);  // -1.5 * 2^23
#pragma unroll
          for (int t = 0; t < DW; t += 2) {
            auto cv = [&](uint32_t x) { return __int_as_float((int)x + 0x4B400000); };
            const float2 f0 = __fadd2_rn(make_float2(cv(d0[t]), cv(d0[t + 1])), mg);
            const float2 f12 = make_float2((float)((int)d1[t] * 256 + (int)d2[t]),
                                           (float)((int)d1[t + 1] * 256 + (int)d2[t + 1]));
            const float2 v = __fmul2_rn(__ffma2_rn(f0, make_float2(65536.0f, 65536.0f), f12),
                                        make_float2(sc[t], sc[t + 1]));
            vv[t] = v.x;
            vv[t + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int t = 0; t < DW; ++t)
            vv[t] = fmaf((float)(int)d0[t], 65536.0f, fmaf((float)(int)d1[t], 256.0f, (float)(int)d2[t])) * sc[t];
        }
        float4* dst = reinterpret_cast<float4*>(&sm.stage[et][g * DW]);
        dst[0] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        dst[1] = make_float4(vv[4], vv[5], vv[6], vv[7]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty);  // the next j-tile's MMAs may start now
      TP_ACC(e_drain, tc0);
      TP_T0(td0);
      // (3) segment sums over this thread's own (sorted) staging row: inclusive prefix sums in
      //     registers, stored back; segment a of chunk c = P[end_a - 1] - P[end_{a-1} - 1]
#pragma unroll 1
      for (int c = 2 * h; c < ((dbg & 1) ? 0 : 2 * h + 2); ++c) {
        float* row = &sm.stage[et][c * 32];
        // this chunk's values in sorted order (the row's permutation, 32 bytes)
        const uint4 pa = reinterpret_cast<const uint4*>(&sm.perm[bf][i][c * 32])[0];
        const uint4 pb = reinterpret_cast<const uint4*>(&sm.perm[bf][i][c * 32])[1];
        const uint32_t pw[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = row[(pw[q >> 2] >> (8 * (q & 3))) & 31];
#pragma unroll
        for (int q = 1; q < 32; ++q) v[q] += v[q - 1];
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          reinterpret_cast<float4*>(row)[q4] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
        uint32_t ow[TcSmem<NLEV>::NLEVP / 4];
#pragma unroll
        for (int w4 = 0; w4 < TcSmem<NLEV>::NLEVP / 4; ++w4)
          ow[w4] = reinterpret_cast<const uint32_t*>(&sm.oend[bf][i][c][0])[w4];
        float lo = 0.0f;
#pragma unroll
        for (int a = 0; a < NLEV; ++a) {
          const int s1 = (ow[a >> 2] >> (8 * (a & 3))) & 0xFF;
          const float hi = (s1 > 0) ? row[s1 - 1] : 0.0f;
          acf[a] += hi - lo;
          lo = hi;
        }
      }
      if ((jt - jt_lo) % FLUSH == FLUSH - 1 || jt + 1 == jt_hi) {
#pragma unroll
        for (int a = 0; a < NLEV; ++a) {
          acc[a] += (double)acf[a];
          acf[a] = 0.0f;
        }
      }
      TP_ACC(e_walk, td0);
    }
    {
      long long tot = 0;
      TP_ACC(tot, t_all);
      tp_flush(dbg, lane, 8, tot);
      tp_flush(dbg, lane, 9, e_sort);
      tp_flush(dbg, lane, 10, e_wait);
      tp_flush(dbg, lane, 11, e_drain);
      tp_flush(dbg, lane, 12, e_walk);
      tp_flush(dbg, lane, 13, e_bar);
    }
    // the two halves' partial sums meet in the (now free) staging tile, in a fixed order
    double* red = reinterpret_cast<double*>(&sm.stage[0][0]);
    named_bar_sync(1, EPI_THREADS);  // every walk has finished with its staging row
    if (h == 1) {
#pragma unroll
      for (int a = 0; a < NLEV; ++a) red[et * NLEV + a] = acc[a];
    }
    named_bar_sync(1, EPI_THREADS);
    const int64_t row = r0 + i;
    if (h == 0 && row < m) {
#pragma unroll
      for (int a = 0; a < NLEV; ++a) Cpart[(row * NLEV + a) * NLEV + b] = acc[a] + red[et * NLEV + a];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
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
  cuuint32_t box[2] = {TK, SLICE};  // 128 k (bytes) x TJ / CS j: one CTA's slice
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)Hq, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(GANQ_ERR_CUDA, "tgram: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GANQ_ERR_CUDA;
  }
  constexpr int R = 128 / NLEV;
  auto kern = tgram_tc_kernel<NLEV>;
  const size_t smem = 1024 + (size_t)stages_of(NLEV) * STAGE_BYTES + sizeof(TcSmem<NLEV>);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // split the j-tiles (work of tile jt = ktiles_of(jt)) into nsplit ranges of equal work
  const int nsplit = tgram_splits(m, NLEV);
  const int NT = (int)((n + TJ - 1) / TJ);
  int64_t total = 0;
  for (int jt = 0; jt < NT; ++jt) total += ktiles_of(jt);
  int bnd[SPLIT - 1] = {NT, NT, NT};
  int64_t acc = 0;
  int jt = 0;
  for (int p = 1; p < nsplit; ++p) {
    while (jt < NT && nsplit * (acc + ktiles_of(jt)) <= p * total) acc += ktiles_of(jt++);
    bnd[p - 1] = jt;
  }
  const int4 jsplit = make_int4(bnd[0], bnd[1], bnd[2], 0);
  const int groups = (int)((m + R - 1) / R);
  const int gp = (groups + CS - 1) / CS * CS;  // whole clusters; extra CTAs own no rows
  static const int dbg = getenv("GANQ_TGRAM_DBG") ? atoi(getenv("GANQ_TGRAM_DBG")) : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nsplit * gp));
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
  GANQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tmap, Q, scale, m, n, P, jsplit, nsplit, gp, Cg, dbg));
  GANQ_LAUNCH_CHECK("tgram_tc_kernel");
  if (dbg & 16) {
    unsigned long long h[16];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_tgprof, sizeof(h));
    const double c = (double)(nsplit * gp);
    fprintf(stderr,
            "tgprof per CTA (kcyc): tma %.1f (wait empty %.1f) | mma %.1f (wait full %.1f, tempty %.1f) | "
            "prod/warp %.1f (wait empty %.1f, st %.1f) | epi/warp %.1f (sort %.1f, wait tfull %.1f, drain %.1f, "
            "walk %.1f, bar %.1f)\n",
            h[0] / c / 1e3, h[1] / c / 1e3, h[2] / c / 1e3, h[3] / c / 1e3, h[4] / c / 1e3, h[5] / c / 4e3,
            h[6] / c / 4e3, h[7] / c / 4e3, h[8] / c / 8e3, h[9] / c / 8e3, h[10] / c / 8e3, h[11] / c / 8e3,
            h[12] / c / 8e3, h[13] / c / 8e3);
    const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_tgprof, z, sizeof(z));
  }
  return GANQ_OK;
}

}  // namespace

int64_t tq_pitch(int64_t n) { return (n + 127) / 128 * 128; }

// CTAs per row group of the normal-matrix kernel = the number of partial C blocks tsolve adds.
// Each CTA carries fixed costs (TMEM allocation, pipeline fill, the last drain and walk), so fewer
// and longer CTAs are better as long as the grid still fills whole waves of 148 SMs: the smallest
// split in 2..4 whose last wave is at least 97 % full, else the fullest (c2: 1024 CTAs in 7 waves;
// measured at c2: 1 / 2 / 3 / 4 ways = 12.3 / 11.1 / 11.7 / 11.6 ms per layer).  GANQ_TGRAM_SPLIT
// overrides it.
int tgram_splits(int64_t m, int nlev) {
  static const int forced = [] {
    const char* e = getenv("GANQ_TGRAM_SPLIT");
    const int v = e ? atoi(e) : 0;
    return v < 0 ? 0 : v > SPLIT ? SPLIT : v;
  }();
  if (forced > 0) return forced;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms = v > 0 ? v : 148;
  }
  const int64_t groups = (m + 128 / nlev - 1) / (128 / nlev);
  const int64_t gp = (groups + CS - 1) / CS * CS;
  int best = SPLIT;
  double best_fill = 0.0;
  for (int s2 = 2; s2 <= SPLIT; ++s2) {
    const double waves = (double)(s2 * gp) / sms;
    const double fill = waves / (double)((int64_t)((s2 * gp + sms - 1) / sms));
    if (fill >= 0.97) return s2;
    if (fill > best_fill) {
      best_fill = fill;
      best = s2;
    }
  }
  return best;
}

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
