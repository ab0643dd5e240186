// sstep.cu -- the S-update: row-parallel back-substitution (Eqs. 15-22, P:178-209;
// Algorithm 1 inner loop), blocked into panels of B = 64 columns.
//
// For row i and column j (n-1 down to 0):
//     z_ij = W_ij + a_ij,   a_ij = sum_{u>j} E_iu * Lhat_uj,   Lhat_uj = L_uj / L_jj   (R-10)
//     Q_ij = argmin_s |z_ij - T_is|   (first index on ties, R-7),   E_ij = W_ij - T_{i,Q_ij}
// (E_iu is the paper's residual r_u.)  The sum over u splits into the columns to the
// right of the current panel (a dense m x B x (n - j1) contraction, "lazy blocked error
// propagation") and the columns inside the panel (sequential, B(B-1)/2 per row).
//
// v1 kernel: one CTA per 32 rows runs the whole sweep (rows are independent, Eq. 2, so
// there is no inter-CTA dependency and one launch per S-update).  Per panel:
//   1. all 8 warps: feedback a = E[rows, j1:] * Lhat[j1:, panel] in fp32 FMA (SIMT),
//   2. warp 0 (lane = row): the 64 sequential decisions with a[] in registers and the
//      64 x 64 diagonal block of Lhat in shared memory (broadcast reads),
//   3. all warps: write Q and E of the panel.
#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int R = 32;    // rows per CTA
constexpr int B = 64;    // panel width
constexpr int UC = 32;   // u-chunk of the feedback contraction
constexpr int THREADS = 256;

// argmin_s |z - t_s| with the first index winning ties, as a balanced tournament
// (left operand = lower indices, replaced only on strict '<').
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

struct Smem {
  float Es[UC][R + 1];     // E chunk, transposed (u, row)
  float Ls[UC][B];         // Lhat[u][panel cols]
  float As[R][B + 1];      // feedback accumulators (row, col)
  float Ws[R][B + 1];      // W panel (row, col)
  float Eo[R][B + 1];      // panel residuals out
  uint8_t Qo[R][B + 4];    // panel codes out
  float Ld[B][B];          // Lhat diagonal block: Ld[c][c'] = Lhat[jb+c][jb+c']
};

template <int NLEV>
__global__ void __launch_bounds__(THREADS, 1)
sstep_kernel(const float* __restrict__ W, const float* __restrict__ Lhat, const float* __restrict__ T,
             int64_t m, int64_t n, uint8_t* __restrict__ Q, float* __restrict__ E) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int fr = tid >> 3;          // feedback row 0..31
  const int fc = (tid & 7) * 8;     // feedback col group

  static_assert(NLEV <= 16, "register-resident codebook");
  // Codebook of the panel warp's row, in registers.
  float t[NLEV];
  if (warp == 0) {
    const int64_t row = r0 + lane;
#pragma unroll
    for (int s = 0; s < NLEV; ++s) t[s] = (row < m) ? T[row * NLEV + s] : 0.0f;
  }

  for (int64_t j1 = n; j1 > 0; j1 -= B) {
    const int64_t jb = j1 - B;  // column of panel slot 0 (negative slots are phantoms)
    // ---- stage W panel and the diagonal block of Lhat
    for (int idx = tid; idx < R * B; idx += THREADS) {
      const int r = idx / B, c = idx % B;
      const int64_t row = r0 + r, j = jb + c;
      sm.Ws[r][c] = (row < m && j >= 0) ? W[row * n + j] : 0.0f;
    }
    for (int idx = tid; idx < B * B; idx += THREADS) {
      const int c = idx / B, c2 = idx % B;
      const int64_t j = jb + c, j2 = jb + c2;
      sm.Ld[c][c2] = (j2 >= 0 && c2 < c) ? Lhat[j * n + j2] : 0.0f;
    }
    // ---- feedback from the columns right of the panel
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
    for (int64_t u0 = j1; u0 < n; u0 += UC) {
      __syncthreads();
      {
        const int r = tid >> 3, uu = (tid & 7) * 4;
        const int64_t row = r0 + r;
#pragma unroll
        for (int q = 0; q < 4; ++q) sm.Es[uu + q][r] = (row < m) ? E[row * n + u0 + uu + q] : 0.0f;
      }
      for (int idx = tid; idx < UC * B; idx += THREADS) {
        const int uu = idx / B, c = idx % B;
        const int64_t j = jb + c;
        sm.Ls[uu][c] = (j >= 0) ? Lhat[(u0 + uu) * n + j] : 0.0f;
      }
      __syncthreads();
#pragma unroll 8
      for (int uu = 0; uu < UC; ++uu) {
        const float e = sm.Es[uu][fr];
        const float4 l0 = *reinterpret_cast<const float4*>(&sm.Ls[uu][fc]);
        const float4 l1 = *reinterpret_cast<const float4*>(&sm.Ls[uu][fc + 4]);
        acc[0] = fmaf(e, l0.x, acc[0]);
        acc[1] = fmaf(e, l0.y, acc[1]);
        acc[2] = fmaf(e, l0.z, acc[2]);
        acc[3] = fmaf(e, l0.w, acc[3]);
        acc[4] = fmaf(e, l1.x, acc[4]);
        acc[5] = fmaf(e, l1.y, acc[5]);
        acc[6] = fmaf(e, l1.z, acc[6]);
        acc[7] = fmaf(e, l1.w, acc[7]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) sm.As[fr][fc + q] = acc[q];
    __syncthreads();
    // ---- sequential panel: warp 0, lane = row
    if (warp == 0) {
      float a[B];
#pragma unroll
      for (int c = 0; c < B; ++c) a[c] = sm.As[lane][c];
#pragma unroll
      for (int c = B - 1; c >= 0; --c) {
        const float w = sm.Ws[lane][c];
        const float z = __fadd_rn(w, a[c]);
        int q;
        float tq;
        argmin_tree<NLEV>(z, t, q, tq);
        const float e = __fsub_rn(w, tq);
        sm.Qo[lane][c] = (uint8_t)q;
        sm.Eo[lane][c] = e;
#pragma unroll
        for (int c2 = 0; c2 < c; ++c2) a[c2] = fmaf(e, sm.Ld[c][c2], a[c2]);
      }
    }
    __syncthreads();
    // ---- write the panel's codes and residuals
    for (int idx = tid; idx < R * B; idx += THREADS) {
      const int r = idx / B, c = idx % B;
      const int64_t row = r0 + r, j = jb + c;
      if (row < m && j >= 0) {
        Q[row * n + j] = sm.Qo[r][c];
        E[row * n + j] = sm.Eo[r][c];
      }
    }
    __syncthreads();
  }
}

template <int NLEV>
ganq_status_t launch_sstep_t(const float* W, const float* Lhat, const float* T, int64_t m, int64_t n,
                             uint8_t* Q, float* E, cudaStream_t st) {
  const size_t smem = sizeof(Smem);
  GANQ_CUDA_TRY(cudaFuncSetAttribute(sstep_kernel<NLEV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  sstep_kernel<NLEV><<<(unsigned)((m + R - 1) / R), THREADS, smem, st>>>(W, Lhat, T, m, n, Q, E);
  GANQ_LAUNCH_CHECK("sstep_kernel");
  return GANQ_OK;
}

}  // namespace

ganq_status_t launch_sstep(const float* W, const float* Lhat, const float* T, int64_t m, int64_t n,
                           int nlev, uint8_t* Q, float* E, cudaStream_t st) {
  switch (nlev) {
    case 2: return launch_sstep_t<2>(W, Lhat, T, m, n, Q, E, st);
    case 4: return launch_sstep_t<4>(W, Lhat, T, m, n, Q, E, st);
    case 8: return launch_sstep_t<8>(W, Lhat, T, m, n, Q, E, st);
    case 16: return launch_sstep_t<16>(W, Lhat, T, m, n, Q, E, st);
    default:
      set_error(GANQ_ERR_INVALID_ARG, "sstep: unsupported number of levels %d", nlev);
      return GANQ_ERR_INVALID_ARG;
  }
}

}  // namespace ganq
