// tstep.cu -- the T-update (Eq. 6; Algorithm 1 "batch update")
//     T_i = W_i H S_i^T (S_i H S_i^T)^dagger      (raw H, reading R-4)
// and the initial codebook T^0 (reading R-6).
//
// Normal matrices G_i = S_i H S_i^T, G_i[a][b] = sum_{j,k} [q_ij=a][q_ik=b] H_jk, are
// built without materialising S_i (one-hot segmented sums): by symmetry
//     G_i = C_i + C_i^T + D_i,   C_i[a][b] = sum_{j>k} [q_ij=a][q_ik=b] H_jk,
//                                D_i[a][a] = sum_j [q_ij=a] H_jj.
// C comes from the tensor-core kernel in tgram_tc.cu; kernel trhs gives D, the right-hand
// side b_i[a] = sum_j [q_ij=a] (W H)_ij and the level counts (one warp per row, fp64).
// Kernel tsolve: one warp per row, Cholesky of the 2^N x 2^N system in fp64
// (unused levels get an identity row -> T = 0, Moore-Penrose, reading R-9); rows whose
// used block is numerically singular fall back to a Jacobi eigen pseudo-inverse.
#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int kTgramSplitMax = 4;  // == SPLIT in tgram_tc.cu; tgram_splits() of them are used

// Per row (one warp): D_i[a] = sum_j [q_ij=a] H_jj, b_i[a] = sum_j [q_ij=a] (W H)_ij and the
// level counts.  Lane l accumulates the columns j = l (mod 32) into its own shared slots
// [level][lane] (no atomics, no per-level selects); the 32 lane partials of each level are then
// added in a fixed order (fp64), so the sums are deterministic.
constexpr int TRHS_WARPS = 4;
template <int NLEV>
__global__ void __launch_bounds__(32 * TRHS_WARPS)
trhs_kernel(const double* __restrict__ hdiag, const float* __restrict__ WH, const uint8_t* __restrict__ Q,
            int64_t m, int64_t n, double* __restrict__ Dv, double* __restrict__ bvec, int* __restrict__ cnt) {
  __shared__ double sD[TRHS_WARPS][NLEV][32], sR[TRHS_WARPS][NLEV][32];
  __shared__ int sC[TRHS_WARPS][NLEV][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * TRHS_WARPS + warp;
  if (row >= m) return;
#pragma unroll
  for (int a = 0; a < NLEV; ++a) {
    sD[warp][a][lane] = 0.0;
    sR[warp][a][lane] = 0.0;
    sC[warp][a][lane] = 0;
  }
  __syncwarp();
  const uint8_t* q = Q + row * n;
  const float* wh = WH + row * n;
  auto add = [&](int a, double hd, float r) {
    if (a < NLEV) {  // codes >= 2^N (only possible through ganq_tstep) belong to no level
      sD[warp][a][lane] += hd;
      sR[warp][a][lane] += (double)r;
      sC[warp][a][lane] += 1;
    }
  };
  // two columns per read-modify-write round: both slots are loaded before either is stored
  // (the chain through shared memory is per pair, not per column); equal codes add in column
  // order, exactly as two successive add() calls
  auto add2 = [&](int a1, double h1, float r1, int a2, double h2, float r2) {
    const bool v1 = a1 < NLEV, v2 = a2 < NLEV, same = a1 == a2;
    const int b1 = v1 ? a1 : 0, b2 = v2 ? a2 : 0;
    double D1 = sD[warp][b1][lane], R1 = sR[warp][b1][lane];
    double D2 = sD[warp][b2][lane], R2 = sR[warp][b2][lane];
    int C1 = sC[warp][b1][lane], C2 = sC[warp][b2][lane];
    if (v1) {
      D1 += h1;
      R1 += (double)r1;
      C1 += 1;
      if (same) {
        D1 += h2;
        R1 += (double)r2;
        C1 += 1;
      }
    }
    if (v2 && !same) {
      D2 += h2;
      R2 += (double)r2;
      C2 += 1;
      sD[warp][b2][lane] = D2;
      sR[warp][b2][lane] = R2;
      sC[warp][b2][lane] = C2;
    }
    if (v1) {
      sD[warp][b1][lane] = D1;
      sR[warp][b1][lane] = R1;
      sC[warp][b1][lane] = C1;
    }
  };
  int64_t j0 = 0;
  if ((n & 3) == 0) {
    // lane takes 4 consecutive columns per 128-column step; two steps of loads in flight
    constexpr int TU = 4;  // 128-column steps with loads in flight together
    for (; j0 + 128 * TU <= n; j0 += 128 * TU) {
      uint32_t qv[TU];
      float4 wv[TU];
      double2 h0[TU], h1[TU];
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const int64_t j = j0 + 128 * u + 4 * lane;
        qv[u] = *reinterpret_cast<const uint32_t*>(q + j);
        wv[u] = *reinterpret_cast<const float4*>(wh + j);
        h0[u] = *reinterpret_cast<const double2*>(hdiag + j);
        h1[u] = *reinterpret_cast<const double2*>(hdiag + j + 2);
      }
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        add2(qv[u] & 255, h0[u].x, wv[u].x, (qv[u] >> 8) & 255, h0[u].y, wv[u].y);
        add2((qv[u] >> 16) & 255, h1[u].x, wv[u].z, qv[u] >> 24, h1[u].y, wv[u].w);
      }
    }
  }
  for (int64_t j = j0 + lane; j < n; j += 32) add(q[j], hdiag[j], wh[j]);
  __syncwarp();
  if (lane < NLEV) {
    double d = 0.0, r = 0.0;
    int c = 0;
    for (int l = 0; l < 32; ++l) {
      d += sD[warp][lane][l];
      r += sR[warp][lane][l];
      c += sC[warp][lane][l];
    }
    Dv[row * NLEV + lane] = d;
    bvec[row * NLEV + lane] = r;
    cnt[row * NLEV + lane] = c;
  }
}

__global__ void hdiag_kernel(const double* __restrict__ H, int64_t n, double* __restrict__ hdiag) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) hdiag[j] = H[j * n + j];
}

// 32 / NLEV rows per warp, each in a segment of NLEV lanes; lane l of a segment holds row l of
// that row's (regularised) 2^N x 2^N system.  Shuffles stay inside the segment (width NLEV).
template <int NLEV>
__global__ void __launch_bounds__(256)
tsolve_kernel(double* __restrict__ G, const double* __restrict__ Dv, const double* __restrict__ bvec,
              const int* __restrict__ cnt, int64_t m, int empty_rule, float* __restrict__ T,
              int* __restrict__ fallback, int nsplit) {
  constexpr int RPW = 32 / NLEV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = lane / NLEV, l = lane % NLEV;
  const int64_t row = ((int64_t)blockIdx.x * 8 + warp) * RPW + seg;
  const bool live = row < m;
  const int64_t rw = live ? row : 0;  // (dead segments compute on row 0 and write nothing)
  const bool used = live && cnt[rw * NLEV + l] > 0;
  auto sh = [](double v, int c) { return __shfl_sync(0xffffffffu, v, c, NLEV); };
  auto shi = [](int v, int c) { return __shfl_sync(0xffffffffu, v, c, NLEV); };
  double g[NLEV];
  double maxdiag = 0.0;
  // assemble G = C + C^T + D; C (strict lower sums j > k) arrives as GANQ_TGRAM_SPLIT
  // partials (j-tile ranges, tgram_tc.cu) stacked along m, added in fixed order.  The warp's
  // RPW rows are contiguous in every partial: coalesced 16-byte loads, all in flight together,
  // summed into shared memory, then read per (l, c) and (c, l)
  __shared__ double sC[8][32 * NLEV];
  const size_t pstride = (size_t)m * NLEV * NLEV;
  {
    const int64_t wrow0 = ((int64_t)blockIdx.x * 8 + warp) * RPW;
    const int64_t nrow = m - wrow0 < RPW ? m - wrow0 : RPW;
    const int total = nrow > 0 ? (int)nrow * NLEV * NLEV : 0;
    const double* src = G + wrow0 * NLEV * NLEV;
#pragma unroll 4
    for (int e = 2 * lane; e < total; e += 64) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < kTgramSplitMax; ++p) {
        if (p >= nsplit) break;
        const double2 v = *reinterpret_cast<const double2*>(src + p * pstride + e);
        acc.x += v.x;
        acc.y += v.y;
      }
      sC[warp][e] = acc.x;
      sC[warp][e + 1] = acc.y;
    }
    __syncwarp();
  }
  const double* cw = &sC[warp][seg * NLEV * NLEV];
#pragma unroll
  for (int c = 0; c < NLEV; ++c) g[c] = cw[l * NLEV + c] + cw[c * NLEV + l] + (c == l ? Dv[rw * NLEV + l] : 0.0);
  __syncwarp();
  if (live) {
#pragma unroll
    for (int c = 0; c < NLEV; ++c) G[(rw * NLEV + l) * NLEV + c] = g[c];  // full G for the pinv path
  }
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const bool usedc = shi(used ? 1 : 0, c) != 0;
    g[c] = (used && usedc) ? g[c] : ((c == l && !used) ? 1.0 : 0.0);
  }
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double d = sh(g[c], c);
    const bool uc = shi(used ? 1 : 0, c) != 0;
    if (uc && d > maxdiag) maxdiag = d;
  }
  double x = used ? bvec[rw * NLEV + l] : 0.0;
  const double tol = (double)NLEV * 2.220446049250313e-16 * maxdiag;
  bool ok = true;
  // Cholesky G = L L^T (lane l keeps row l of L in g[0..l])
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double piv = sh(g[c], c);
    if (!(piv > tol)) ok = false;
    const double lcc = sqrt(piv > 0.0 ? piv : 1.0);
    const double lic = (l > c) ? g[c] / lcc : (l == c ? lcc : 0.0);
    g[c] = lic;
#pragma unroll
    for (int q = c + 1; q < NLEV; ++q) {
      const double lqc = sh(lic, q);
      if (l > c && q <= l) g[q] -= lic * lqc;
    }
  }
  // forward: L y = b
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double lcc = sh(g[c], c);
    const double yc = sh(x, c) / lcc;
    if (l == c) x = yc;
    else if (l > c) x -= g[c] * yc;
  }
  // backward: L^T t = y  (L^T row c = column c of L: lane q holds L[q][c] in g[c])
#pragma unroll
  for (int c = NLEV - 1; c >= 0; --c) {
    const double lcc = sh(g[c], c);
    const double tc = sh(x, c) / lcc;
    if (l == c) x = tc;
    // x_r -= L[c][r] * t_c for r < c : lane c holds L[c][r] = g[r]; broadcast per r
#pragma unroll
    for (int r = 0; r < c; ++r) {
      const double lcr = sh(g[r], c);
      if (l == r) x -= lcr * tc;
    }
  }
  // the segment's rows are all usable, else its row takes the pseudo-inverse path
  const unsigned bad = __ballot_sync(0xffffffffu, !ok);
  const unsigned segmask = (NLEV == 32 ? 0xffffffffu : ((1u << NLEV) - 1u)) << (seg * NLEV);
  if (!live) return;
  if (bad & segmask) {
    if (l == 0) fallback[row] = 1;
    return;
  }
  float out = (float)x;
  if (!used) out = (empty_rule == 1) ? T[row * NLEV + l] : 0.0f;
  T[row * NLEV + l] = out;
}

// Rare path: Moore-Penrose by cyclic Jacobi (one thread per flagged row, fp64).
template <int NLEV>
__global__ void tsolve_pinv_kernel(const double* __restrict__ G, const double* __restrict__ bvec,
                                   const int* __restrict__ cnt, int64_t m, int empty_rule,
                                   float* __restrict__ T, int* __restrict__ fallback) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m || !fallback[row]) return;
  double A[NLEV][NLEV], V[NLEV][NLEV];
  for (int i = 0; i < NLEV; ++i)
    for (int j = 0; j < NLEV; ++j) {
      A[i][j] = G[(row * NLEV + i) * NLEV + j];
      V[i][j] = (i == j) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < NLEV; ++i)
      for (int j = 0; j < NLEV; ++j) {
        tot += A[i][j] * A[i][j];
        if (i != j) off += A[i][j] * A[i][j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < NLEV - 1; ++p)
      for (int r = p + 1; r < NLEV; ++r) {
        const double apq = A[p][r];
        if (apq == 0.0) continue;
        const double theta = (A[r][r] - A[p][p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < NLEV; ++k) {
          const double akp = A[k][p], akq = A[k][r];
          A[k][p] = c * akp - s * akq;
          A[k][r] = s * akp + c * akq;
        }
        for (int k = 0; k < NLEV; ++k) {
          const double apk = A[p][k], aqk = A[r][k];
          A[p][k] = c * apk - s * aqk;
          A[r][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < NLEV; ++k) {
          const double vkp = V[k][p], vkq = V[k][r];
          V[k][p] = c * vkp - s * vkq;
          V[k][r] = s * vkp + c * vkq;
        }
      }
  }
  double lmax = 0.0;
  for (int k = 0; k < NLEV; ++k) lmax = fmax(lmax, fabs(A[k][k]));
  const double cut = (double)NLEV * 2.220446049250313e-16 * lmax;
  double x[NLEV];
  for (int a = 0; a < NLEV; ++a) x[a] = 0.0;
  for (int k = 0; k < NLEV; ++k) {
    const double lam = A[k][k];
    if (!(lam > cut)) continue;
    double proj = 0.0;
    for (int a = 0; a < NLEV; ++a) proj += bvec[row * NLEV + a] * V[a][k];
    proj /= lam;
    for (int a = 0; a < NLEV; ++a) x[a] += proj * V[a][k];
  }
  for (int a = 0; a < NLEV; ++a) {
    const bool used = cnt[row * NLEV + a] > 0;
    T[row * NLEV + a] = used ? (float)x[a] : (empty_rule == 1 ? T[row * NLEV + a] : 0.0f);
  }
  fallback[row] = 0;
}

// T^0: per-row fp32 min-max grid (reading R-6): step = (max - min) / (2^N - 1),
// t_s = min + s * step, each operation rounded to fp32 (no FMA contraction).
__global__ void init_codebook_kernel(const float* __restrict__ W, int64_t m, int64_t n, int nlev,
                                     float* __restrict__ T) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const float* w = W + row * n;
  float mn = w[0], mx = w[0];
  for (int64_t j = lane; j < n; j += 32) {
    mn = fminf(mn, w[j]);
    mx = fmaxf(mx, w[j]);
  }
  for (int o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const float step = __fdiv_rn(__fsub_rn(mx, mn), (float)(nlev - 1));
  for (int s = lane; s < nlev; s += 32) T[row * nlev + s] = __fadd_rn(mn, __fmul_rn((float)s, step));
}

template <int NLEV>
ganq_status_t launch_tsolve_t(const double* hdiag, const float* WH, const uint8_t* Q, int64_t m, int64_t n,
                              int empty_rule, float* T, double* G, double* Dv, double* b, int* cnt, int* fb,
                              cudaStream_t st) {
  trhs_kernel<NLEV><<<(unsigned)((m + TRHS_WARPS - 1) / TRHS_WARPS), 32 * TRHS_WARPS, 0, st>>>(hdiag, WH, Q, m, n,
                                                                                               Dv, b, cnt);
  GANQ_LAUNCH_CHECK("trhs_kernel");
  tsolve_kernel<NLEV><<<(unsigned)((m + 8 * (32 / NLEV) - 1) / (8 * (32 / NLEV))), 256, 0, st>>>(G, Dv, b, cnt, m,
                                                                                           empty_rule, T, fb,
                                                                                           tgram_splits(m, NLEV));
  GANQ_LAUNCH_CHECK("tsolve_kernel");
  tsolve_pinv_kernel<NLEV><<<(unsigned)((m + 127) / 128), 128, 0, st>>>(G, b, cnt, m, empty_rule, T,
                                                                         fb);
  GANQ_LAUNCH_CHECK("tsolve_pinv_kernel");
  return GANQ_OK;
}

}  // namespace

ganq_status_t launch_init_codebook(const float* W, int64_t m, int64_t n, int nlev, float* T,
                                   cudaStream_t st) {
  init_codebook_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(W, m, n, nlev, T);
  GANQ_LAUNCH_CHECK("init_codebook_kernel");
  return GANQ_OK;
}

ganq_status_t launch_hdiag(const double* H, int64_t n, double* hdiag, cudaStream_t st) {
  hdiag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(H, n, hdiag);
  GANQ_LAUNCH_CHECK("hdiag_kernel");
  return GANQ_OK;
}

ganq_status_t launch_tsolve(const double* hdiag, const float* WH, const uint8_t* Q, int64_t m, int64_t n, int nlev,
                            int empty_rule, float* T, double* G, double* Dv, double* b, int* cnt, int* fb,
                            cudaStream_t st) {
  switch (nlev) {
    case 2: return launch_tsolve_t<2>(hdiag, WH, Q, m, n, empty_rule, T, G, Dv, b, cnt, fb, st);
    case 4: return launch_tsolve_t<4>(hdiag, WH, Q, m, n, empty_rule, T, G, Dv, b, cnt, fb, st);
    case 8: return launch_tsolve_t<8>(hdiag, WH, Q, m, n, empty_rule, T, G, Dv, b, cnt, fb, st);
    case 16: return launch_tsolve_t<16>(hdiag, WH, Q, m, n, empty_rule, T, G, Dv, b, cnt, fb, st);
    default:
      set_error(GANQ_ERR_UNSUPPORTED, "tsolve: 2^N = %d levels unsupported (N must be 1..4)", nlev);
      return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
