// cholesky.cu -- preconditioning (App. A Eqs. 23-24; Remark 1),
// the fp64 Cholesky factor H' = L L^T (Eq. 9; Algorithm 1), and the
// fp32 operands the S- and T-updates read (reading R-10).
//
// Factorisation: right-looking blocked Cholesky with NB = 64, in place on the lower
// triangle of A (fp64).  Per block column k: (1) one launch factors the 64 x 64 diagonal
// block and solves the panel below it (every CTA eliminates the diagonal block plus 64 panel
// rows in registers), (2) trailing SYRK update of the lower tiles (128 x 128
// tiles, 8 x 8 fp64 register blocking), applied once per two panels (K = 128).  Each tile has
// one owner per step, so the result is deterministic (bitwise identical on every rank).
// A non-positive pivot records its global index (atomicMin) in *d_status.
#include <float.h>
#include <stdlib.h>
#include <limits.h>

#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int NB = 64;
constexpr int LDS = NB + 1;  // padded fp64 row stride in shared memory

// 8-byte global -> shared copy that does not hold a register (all of a tile's copies are in
// flight together; cp_wait() before the barrier that publishes them)
__device__ __forceinline__ void cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------- precondition
// delta_i = max(sum_j |H_ij| - 2 H_ii, 1e-8) + tau * mean(diag H)   (ADAPTIVE, Eq. 23 + R-3)
// delta_i = lambda                                                  (FIXED_LAMBDA)
// delta_i = 0                                                        (NONE)
__global__ void diag_mean_kernel(const double* __restrict__ H, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += H[i * n + i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s / (double)n;
  }
}

// One warp per row: A = H (full row copy) with A_ii += delta_i.
__global__ void precondition_kernel(const double* __restrict__ H, int64_t n, int policy,
                                    double lambda, double tau, const double* __restrict__ diag_mean,
                                    double* __restrict__ A, double* __restrict__ delta) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double* h = H + i * n;
  double* a = A + i * n;
  double rs = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    const double v = h[j];
    a[j] = v;
    rs += fabs(v);
  }
  for (int o = 16; o; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  if (lane == 0) {
    double d = 0.0;
    if (policy == GANQ_PRECOND_ADAPTIVE) {
      d = rs - 2.0 * h[i];
      if (d < 1e-8) d = 1e-8;
      d += tau * (*diag_mean);
    } else if (policy == GANQ_PRECOND_FIXED_LAMBDA) {
      d = lambda;
    }
    a[i] = h[i] + d;
    if (delta) delta[i] = d;
  }
}

// ---------------------------------------------------------------- panel factor (POTRF + TRSM)
// Block column k0 (kb <= 64 columns) of the right-looking factorisation, restricted to its own
// columns: every CTA holds the 64 x 64 diagonal block plus PR rows of the panel below it and
// runs the unscaled elimination on those 128 rows -- step c subtracts a_rc a_qc / d_c from the
// elements right of column c (d_c = a_cc, the pivot), which for the panel rows is exactly the
// forward substitution x L_kk^T = A_panel and for the diagonal block the Cholesky of L_kk;
// afterwards L_rc = a_rc / sqrt(d_c).  The diagonal block is factored redundantly by every
// CTA (same instructions, same result), so POTRF and TRSM are one launch whose dependent chain
// is 64 column steps of {one barrier, one broadcast read of column c, 32 FMAs per thread}.
// Thread (tx, ty) keeps its 8 x 4 elements (ty + 16 a, tx + 16 b) in registers; the owners of
// column c publish it to shared memory (double-buffered, one barrier per step).  The CTA that
// finishes last writes the diagonal block (every other CTA has read its input by then -- CTAs
// of a large grid, or ones delayed behind another stream's kernel, start late); a non-positive
// pivot records its global index in *status.
constexpr int PR = 64;          // panel rows per CTA
constexpr int PROWS = NB + PR;  // rows held per CTA
constexpr int PF_THREADS = 256; // thread (tx, ty): rows ty + 16 a (a < 8), columns tx + 16 b (b < 4)
// 1 / d to ~1 ulp: hardware estimate + two Newton steps (no slow-path branch on the chain)
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = r * fma(-d, r, 2.0);
  return r * fma(-d, r, 2.0);
}
__global__ void __launch_bounds__(PF_THREADS) panel_factor_kernel(double* __restrict__ A, int64_t n, int64_t k0,
                                                                  int* __restrict__ status, int* __restrict__ ticket) {
  __shared__ double col[2 * PROWS];  // column c of the 128 rows, double-buffered
  __shared__ double dpiv[NB];
  __shared__ int last;
  const int kb = (int)min((int64_t)NB, n - k0);
  const int64_t p0 = k0 + kb + (int64_t)blockIdx.x * PR;  // first panel row of this CTA
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  // element (ty + 16 a, tx + 16 b); a < 4: the diagonal block, a >= 4: panel rows
  double v[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, q = tx + 16 * b;
      if (a < NB / 16) {
        v[a][b] = (r < kb && q <= r) ? A[(k0 + r) * n + k0 + q] : (r == q ? 1.0 : 0.0);
      } else {
        const int64_t i = p0 + (r - NB);
        v[a][b] = (i < n && q < kb) ? A[i * n + k0 + q] : 0.0;
      }
    }
  // Column c = 16 bc + cl: its owners are the threads with tx == cl (register slot b = bc, a
  // compile-time index).  Step c updates (r, q) with r > c and q > c: column blocks b < bc are
  // final and skipped, block bc is masked by q > c, diagonal-block rows by r > c.
#pragma unroll
  for (int bc = 0; bc < 4; ++bc) {
#pragma unroll 1
    for (int cl = 0; cl < 16; ++cl) {
      const int c = 16 * bc + cl;
      const int buf = (c & 1) * PROWS;
      if (tx == cl) {
#pragma unroll
        for (int a = 0; a < 8; ++a) col[buf + ty + 16 * a] = v[a][bc];
      }
      __syncthreads();
      double d = col[buf + c];
      double cr[8], cq[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) cr[a] = (a >= NB / 16 || ty + 16 * a > c) ? col[buf + ty + 16 * a] : 0.0;
#pragma unroll
      for (int b = bc; b < 4; ++b) cq[b] = (b > bc || tx > cl) ? col[buf + tx + 16 * b] : 0.0;
      if (!(d > 0.0)) {  // not positive definite (or NaN)
        if (threadIdx.x == 0 && blockIdx.x == 0 && c < kb) atomicMin(status, (int)(k0 + c));
        d = 1.0;
      }
      if (threadIdx.x == 0) dpiv[c] = d;
      const double id = rcp_nr(d);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const double t = cr[a] * id;
#pragma unroll
        for (int b = bc; b < 4; ++b) v[a][b] = fma(-t, cq[b], v[a][b]);
      }
    }
  }
  __syncthreads();
  // L_rq = a_rq / sqrt(d_q), L_qq = sqrt(d_q)
  double sd[4], isd[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    sd[b] = sqrt(dpiv[tx + 16 * b]);
    isd[b] = 1.0 / sd[b];
  }
#pragma unroll
  for (int a = NB / 16; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, q = tx + 16 * b;
      const int64_t i = p0 + (r - NB);
      if (i < n && q < kb) A[i * n + k0 + q] = v[a][b] * isd[b];
    }
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!last) return;
#pragma unroll
  for (int a = 0; a < NB / 16; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = ty + 16 * a, q = tx + 16 * b;
      if (r < kb && q <= r) A[(k0 + r) * n + k0 + q] = (q == r) ? sd[b] : v[a][b] * isd[b];
    }
  if (threadIdx.x == 0) *ticket = 0;  // ready for the next panel launch (stream-ordered)
}

// ---------------------------------------------------------------- trailing SYRK
// A[i, j] -= sum_{c in [k0, k0 + kw)} L[i, c] L[j, c] for base <= j <= i < n, j < cend: the lower
// 128 x 128 tiles of the trailing block.  Persistent CTAs (one per SM) walk the tile list; the
// panel columns stream through shared memory in chunks of KC = 32 with the next chunk's
// cp.async copies (possibly the next tile's) in flight while the current chunk is multiplied.
// The products run on the fp64 tensor cores (DMMA m8n8k4, 256 FMAs per warp instruction; the
// same 37 TF/s as the FMA pipe, but without the operand traffic that held an 8 x 8 register
// outer product to ~45 %): 8 warps of 64 x 32 each, fp64 accumulators in registers.  The tile
// is subtracted with fire-and-forget L2 reductions (RED.ADD.F64): every element has one owner
// per launch and launches are stream-ordered, so this equals a read-modify-write bit for bit.
constexpr int ST = 128;       // SYRK tile
constexpr int KC = 32;        // panel columns per chunk
constexpr int PLD = KC + 4;   // fp64 row stride of a staged chunk: fragment loads conflict-free
// shared memory: 2 buffers x (TI + TJ) rows x PLD
constexpr int SYRK_SMEM_THIN = 2 * 2 * 64 * PLD * (int)sizeof(double);  // 64 x 64
constexpr int SYRK_SMEM_BULK = 2 * (ST + 64) * PLD * (int)sizeof(double);  // 128 x 64

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct SyrkTiles {  // lower tiles in row-major order: row ti holds j-tiles tj < min(R (ti + 1), Tj)
  int Ti, Tj, R;     // R = TI / TJ (1 or 2)
  __host__ __device__ int tri_rows() const { return (Tj + R - 1) / R - 1; }  // rows with < Tj tiles
  __host__ __device__ int cum(int r) const { return R * r * (r + 1) / 2; }  // tiles in rows < r (r <= tri_rows)
  __host__ __device__ int count() const {
    const int rt = Ti < tri_rows() ? Ti : tri_rows();
    return cum(rt) + (Ti > rt ? (Ti - rt) * Tj : 0);
  }
  __device__ void at(int t, int& ti, int& tj) const {
    const int rt = Ti < tri_rows() ? Ti : tri_rows();
    if (t < cum(rt)) {
      int r = (int)((sqrtf(8.0f * (float)t / (float)R + 1.0f) - 1.0f) * 0.5f);
      while (r > 0 && cum(r) > t) --r;
      while (cum(r + 1) <= t) ++r;
      ti = r;
      tj = t - cum(r);
    } else {
      const int u = t - cum(rt);
      ti = rt + u / Tj;
      tj = u % Tj;
    }
  }
};

// TI x TJ tiles (128 x 128 for the bulk update; 64 x 64 for the thin update of the next panel's
// 64 columns, twice the CTAs and none of the masked half-tile work); 8 warps as 2 (rows) x 4
// (columns), each TI/2 x TJ/4 = MB x NBB blocks of 8 x 8.
template <int TI, int TJ>
__global__ void __launch_bounds__(256, TJ < 128 ? 2 : 1) syrk_trailing_kernel(double* __restrict__ A, int64_t n, int64_t k0,
                                                               int kw, int64_t base, int64_t cend,
                                                               SyrkTiles tl) {
  constexpr int MB = TI / 16, NBB = TJ / 32;
  constexpr int BUF = (TI + TJ) * PLD;  // one buffer: rows i, then rows j
  extern __shared__ double syrk_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 1, wn = warp >> 1;  // warp tile: rows (TI/2) wm + [0, TI/2), cols (TJ/4) wn + ...
  const int gr = lane >> 2, gk = lane & 3;  // fragment row / k (A, B) and row / column pair (C)
  const int ntiles = tl.count();
  const int nch = (kw + KC - 1) / KC;
  const int mytiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = mytiles * nch;  // this CTA's chunk sequence: (tile u, chunk kc)
  // stage chunk g of the sequence into buffer g & 1 (16-byte copies when rows allow: n even,
  // k0 even; else 8-byte copies)
  const bool vec = ((n | k0) & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  auto issue = [&](int g) {
    const int u = g / nch, kc = (g % nch) * KC;
    int ti, tj;
    tl.at((int)blockIdx.x + u * (int)gridDim.x, ti, tj);
    const int64_t i0 = base + (int64_t)ti * TI, j0 = base + (int64_t)tj * TJ;
    const int kcw = min(KC, kw - kc);
    double* Pi = syrk_smem + (g & 1) * BUF;
    double* Pj = Pi + TI * PLD;
    if (vec && kcw == KC) {
#pragma unroll 1
      for (int e = threadIdx.x; e < TI * KC / 2; e += 256) {
        const int r = e >> 4, c = (e & 15) * 2;
        if (i0 + r < n) cp16(&Pi[r * PLD + c], &A[(i0 + r) * n + k0 + kc + c]);
        else *reinterpret_cast<double2*>(&Pi[r * PLD + c]) = make_double2(0.0, 0.0);
      }
#pragma unroll 1
      for (int e = threadIdx.x; e < TJ * KC / 2; e += 256) {
        const int r = e >> 4, c = (e & 15) * 2;
        if (j0 + r < cend) cp16(&Pj[r * PLD + c], &A[(j0 + r) * n + k0 + kc + c]);
        else *reinterpret_cast<double2*>(&Pj[r * PLD + c]) = make_double2(0.0, 0.0);
      }
    } else {
      for (int e = threadIdx.x; e < (TI + TJ) * KC; e += 256) {
        const int r = e / KC, c = e % KC;
        const bool isi = r < TI;
        const int rr = isi ? r : r - TI;
        const int64_t gr0 = isi ? i0 + rr : j0 + rr;
        double* dst = (isi ? Pi : Pj) + rr * PLD + c;
        if (gr0 < (isi ? n : cend) && c < kcw) cp8(dst, &A[gr0 * n + k0 + kc + c]);
        else *dst = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[MB][NBB][2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NBB; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
  if (total > 0) issue(0);
  for (int g = 0; g < total; ++g) {
    if (g + 1 < total) {
      issue(g + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* Pi = syrk_smem + (g & 1) * BUF + ((TI / 2) * wm + gr) * PLD + gk;
    const double* Pj = syrk_smem + (g & 1) * BUF + TI * PLD + ((TJ / 4) * wn + gr) * PLD + gk;
#pragma unroll 2
    for (int ks = 0; ks < KC; ks += 4) {
      double a[MB], b[NBB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) a[mb] = Pi[mb * 8 * PLD + ks];
#pragma unroll
      for (int nb = 0; nb < NBB; ++nb) b[nb] = Pj[nb * 8 * PLD + ks];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NBB; ++nb) dmma884(acc[mb][nb], a[mb], b[nb]);
    }
    if (g % nch == nch - 1) {
      int ti, tj;
      tl.at((int)blockIdx.x + (g / nch) * (int)gridDim.x, ti, tj);
      const int64_t t_i0 = base + (int64_t)ti * TI, t_j0 = base + (int64_t)tj * TJ;
      const int64_t i0 = t_i0 + (TI / 2) * wm + gr, j0 = t_j0 + (TJ / 4) * wn + 2 * gk;
      const bool interior = t_i0 >= t_j0 + TJ && t_i0 + TI <= n && t_j0 + TJ <= cend;
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        const int64_t i = i0 + 8 * mb;
        double* row = A + i * n + j0;
#pragma unroll
        for (int nb = 0; nb < NBB; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t j = j0 + 8 * nb + h;
            if (interior || (i < n && j <= i && j < cend)) atomicAdd(row + 8 * nb + h, -acc[mb][nb][h]);
            acc[mb][nb][h] = 0.0;
          }
      }
    }
    __syncthreads();  // buffer g & 1 is free for chunk g + 2
  }
}

__global__ void zero_upper_kernel(double* __restrict__ A, int64_t n) {
  const int64_t total = n * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx % n;
    if (j > i) A[idx] = 0.0;
  }
}

// ---------------------------------------------------------------- derived fp32 operands
// Lhat[u][j] = L_uj / L_jj for u > j, 0 otherwise (the S-update's scaled feedback
// weights, reading R-10); H32 = fp32(H) for the T-update (reading R-4: raw H).
__global__ void derive_kernel(const double* __restrict__ L, const double* __restrict__ H, int64_t n,
                              float* __restrict__ Lhat, float* __restrict__ H32) {
  const int64_t total = n * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = idx / n, j = idx % n;
    if (Lhat) Lhat[idx] = (u > j) ? (float)(L[idx] / L[j * n + j]) : 0.0f;
    if (H32) H32[idx] = (float)H[idx];
  }
}

}  // namespace

ganq_status_t launch_precondition(const double* H, int64_t n, int policy, double lambda, double tau,
                                  double* A, double* delta, double* d_mean, cudaStream_t st) {
  diag_mean_kernel<<<1, 1024, 0, st>>>(H, n, d_mean);
  GANQ_LAUNCH_CHECK("diag_mean_kernel");
  precondition_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(H, n, policy, lambda, tau, d_mean, A,
                                                               delta);
  GANQ_LAUNCH_CHECK("precondition_kernel");
  return GANQ_OK;
}

// Side stream and events of the Cholesky look-ahead, created once per host thread and device.
struct LookAhead {
  int device = -1;
  cudaStream_t side = nullptr;
  cudaEvent_t th = nullptr, tr = nullptr;
};
LookAhead& look_ahead() {
  static thread_local LookAhead la;
  int dev = 0;
  cudaGetDevice(&dev);
  if (la.device != dev) {
    // highest priority: the side stream's panel kernels take SMs as soon as bulk-update CTAs
    // retire instead of queueing behind the bulk kernel's remaining CTAs
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&la.side, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&la.th, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&la.tr, cudaEventDisableTiming);
    la.device = dev;
  }
  return la;
}

namespace {
// The blocked factorisation's launch sequence on `st` (plus the look-ahead side stream).
ganq_status_t enqueue_cholesky(double* A, int64_t n, int* d_status, int* d_ticket, cudaStream_t st) {
  auto panel = [&](int64_t k0, cudaStream_t ps) -> ganq_status_t {
    const int64_t rest = n - k0 - NB;
    const unsigned grid = rest > 0 ? (unsigned)((rest + PR - 1) / PR) : 1u;
    panel_factor_kernel<<<grid, PF_THREADS, 0, ps>>>(A, n, k0, d_status, d_ticket);
    GANQ_LAUNCH_CHECK("panel_factor_kernel");
    return GANQ_OK;
  };
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  auto syrk = [&](int64_t k0, int kw, int64_t base, int64_t cend) -> ganq_status_t {
    SyrkTiles tl;
    if (cend - base <= 64 && (n - base + 63) / 64 <= sms) {  // thin: the next panel's 64 columns, one wave
      tl.Ti = (int)((n - base + 63) / 64);
      tl.Tj = 1;
      tl.R = 1;
      syrk_trailing_kernel<64, 64><<<(unsigned)min(tl.Ti, sms), 256, SYRK_SMEM_THIN, st>>>(A, n, k0, kw, base,
                                                                                         cend, tl);
    } else {
      // 128 x 64 tiles, two CTAs per SM: one CTA's loads and reductions overlap the other's MMAs
      tl.Ti = (int)((n - base + ST - 1) / ST);
      tl.Tj = (int)((cend - base + 63) / 64);
      tl.R = 2;
      syrk_trailing_kernel<ST, 64><<<(unsigned)min(tl.count(), 2 * sms), 256, SYRK_SMEM_BULK, st>>>(
          A, n, k0, kw, base, cend, tl);
    }
    GANQ_LAUNCH_CHECK("syrk_trailing_kernel");
    return GANQ_OK;
  };
  if (n < 6144) {
    // One panel per pass with look-ahead: the trailing update of panel k is split into a thin
    // update of panel k+1's columns and the bulk (columns beyond); panel k+1's diagonal factor
    // and TRSM run on a side stream while the bulk update of panel k runs on `st`.
    //   side:  potrf(k+1), trsm(k+1)    after thin(k)          (event th)
    //   st:    thin(k+1)                after trsm(k+1)        (event tr)
    // thin(k) follows bulk(k-1) on st, so panel k+1 has every earlier update when it starts.
    LookAhead& la = look_ahead();
    GANQ_CUDA_TRY(cudaEventRecord(la.th, st));
    GANQ_CUDA_TRY(cudaStreamWaitEvent(la.side, la.th, 0));
    ganq_status_t s;
    if ((s = panel(0, la.side))) return s;
    GANQ_CUDA_TRY(cudaEventRecord(la.tr, la.side));
    for (int64_t k0 = 0; k0 < n; k0 += NB) {
      const int64_t k1 = k0 + NB;
      if (k1 >= n) break;
      GANQ_CUDA_TRY(cudaStreamWaitEvent(st, la.tr, 0));  // trsm(k) done
      if ((s = syrk(k0, NB, k1, min(k1 + NB, n)))) return s;  // thin(k): panel k+1's columns
      GANQ_CUDA_TRY(cudaEventRecord(la.th, st));
      GANQ_CUDA_TRY(cudaStreamWaitEvent(la.side, la.th, 0));
      if ((s = panel(k1, la.side))) return s;                // overlaps bulk(k) below
      GANQ_CUDA_TRY(cudaEventRecord(la.tr, la.side));
      if (k1 + NB < n)
        if ((s = syrk(k0, NB, k1 + NB, n))) return s;        // bulk(k)
    }
    GANQ_CUDA_TRY(cudaStreamWaitEvent(st, la.tr, 0));      // the last panel is factored
  } else {
    // large n: two panels per pass -- factor panel k, update only panel k + 1's columns (thin
    // SYRK), factor panel k + 1, then one trailing SYRK with both panels (K = 128): the trailing
    // matrix (beyond L2) is read and written once per 128 columns.  (Look-ahead on the side
    // stream was measured slower here: the HBM-bound bulk update loses SMs to the panel kernels.)
    for (int64_t k0 = 0; k0 < n; k0 += 2 * NB) {
      ganq_status_t s;
      if ((s = panel(k0, st))) return s;
      const int64_t k1 = k0 + NB;
      if (k1 >= n) break;
      if ((s = syrk(k0, NB, k1, min(k1 + NB, n)))) return s;  // panel k+1's columns only
      if ((s = panel(k1, st))) return s;
      const int64_t base = k1 + NB;
      if (base >= n) break;
      if ((s = syrk(k0, 2 * NB, base, n))) return s;          // trailing block, both panels
    }
  }
  zero_upper_kernel<<<1184, 256, 0, st>>>(A, n);
  GANQ_LAUNCH_CHECK("zero_upper_kernel");
  return GANQ_OK;
}

// The look-ahead sequence (n < 6144: ~190 launches and ~130 cross-stream event hops) captured
// once per (A, n, status, ticket, device) into a CUDA graph and replayed on a private stream
// forked from / joined to the caller's stream; GANQ_CHOL_GRAPH=0 launches it directly.
struct CholGraph {
  int device = -1;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t exec = nullptr;
  double* A = nullptr;
  int64_t n = 0;
  int *status = nullptr, *ticket = nullptr;
  unsigned long long nlaunch = 0;
};
CholGraph& chol_graph() {
  static thread_local CholGraph g;
  return g;
}
}  // namespace

ganq_status_t launch_cholesky(double* A, int64_t n, int* d_status, int* d_ticket, cudaStream_t st) {
  GANQ_CUDA_TRY(cudaFuncSetAttribute(syrk_trailing_kernel<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SYRK_SMEM_THIN));
  GANQ_CUDA_TRY(cudaFuncSetAttribute(syrk_trailing_kernel<ST, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SYRK_SMEM_BULK));
  static const bool use_graph = !getenv("GANQ_CHOL_GRAPH") || atoi(getenv("GANQ_CHOL_GRAPH")) != 0;
  if (!use_graph || n >= 6144) return enqueue_cholesky(A, n, d_status, d_ticket, st);
  CholGraph& g = chol_graph();
  int dev = 0;
  GANQ_CUDA_TRY(cudaGetDevice(&dev));
  if (g.device != dev) {
    g = CholGraph();
    // high priority: the factorisation's panel chain takes SMs ahead of work overlapping it
    int lo = 0, hi = 0;
    GANQ_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GANQ_CUDA_TRY(cudaStreamCreateWithPriority(&g.cs, cudaStreamNonBlocking, hi));
    GANQ_CUDA_TRY(cudaEventCreateWithFlags(&g.ev_in, cudaEventDisableTiming));
    GANQ_CUDA_TRY(cudaEventCreateWithFlags(&g.ev_out, cudaEventDisableTiming));
    g.device = dev;
  }
  // fork: the private stream waits for the caller's stream (status / ticket initialised there)
  GANQ_CUDA_TRY(cudaEventRecord(g.ev_in, st));
  GANQ_CUDA_TRY(cudaStreamWaitEvent(g.cs, g.ev_in, 0));
  if (!(g.exec && g.A == A && g.n == n && g.status == d_status && g.ticket == d_ticket)) {
    if (g.exec) {
      GANQ_CUDA_TRY(cudaGraphExecDestroy(g.exec));
      g.exec = nullptr;
    }
    const unsigned long long c0 = ganq_launch_count();
    GANQ_CUDA_TRY(cudaStreamBeginCapture(g.cs, cudaStreamCaptureModeThreadLocal));
    const ganq_status_t s = enqueue_cholesky(A, n, d_status, d_ticket, g.cs);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(g.cs, &graph);
    if (s) {
      if (graph) cudaGraphDestroy(graph);
      return s;
    }
    GANQ_CUDA_TRY(e);
    const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    GANQ_CUDA_TRY(ei);
    g.nlaunch = ganq_launch_count() - c0;  // kernels recorded (counted once, at capture)
    g.A = A;
    g.n = n;
    g.status = d_status;
    g.ticket = d_ticket;
  } else {
    for (unsigned long long i = 0; i < g.nlaunch; ++i) count_launch();
  }
  GANQ_CUDA_TRY(cudaGraphLaunch(g.exec, g.cs));
  // join: the caller's stream continues after the factorisation
  GANQ_CUDA_TRY(cudaEventRecord(g.ev_out, g.cs));
  GANQ_CUDA_TRY(cudaStreamWaitEvent(st, g.ev_out, 0));
  return GANQ_OK;
}

ganq_status_t launch_derive_operands(const double* L, const double* H, int64_t n, float* Lhat,
                                     float* H32, cudaStream_t st) {
  derive_kernel<<<1184, 256, 0, st>>>(L, H, n, Lhat, H32);
  GANQ_LAUNCH_CHECK("derive_kernel");
  return GANQ_OK;
}

}  // namespace ganq
