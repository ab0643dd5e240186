// tstep.cu -- the T-update (Eq. 6; Algorithm 1 "batch update")
//     T_i = W_i H S_i^T (S_i H S_i^T)^dagger      (raw H, reading R-4)
// and the initial codebook T^0 (reading R-6).
//
// Normal matrices G_i = S_i H S_i^T, G_i[a][b] = sum_{j,k} [q_ij=a][q_ik=b] H_jk, are
// built without materialising S_i (one-hot segmented sums): by symmetry
//     G_i = C_i + C_i^T + D_i,   C_i[a][b] = sum_{j>k} [q_ij=a][q_ik=b] H_jk,
//                                D_i[a][a] = sum_j [q_ij=a] H_jj.
// Kernel tgram: one warp per row, 8 rows per CTA sharing 32 x 128 tiles of H (fp32,
// strict lower part) staged in shared memory.  Lanes own 4 consecutive columns k
// (float4); for each level a the warp walks the j's of the tile whose code is a
// (ballot mask, warp-uniform), so a sits in a static register index: acc[a][v] += H[j][k_v].
// After a 128-column chunk, acc[a][v] is scattered to the bin b_v = q_ik by a
// deterministic shuffle reduction into fp64 accumulators (no atomics: bitwise
// reproducible).  RHS b_i[a] = sum_j [q_ij=a] (W H)_ij and the level counts come from the
// same kernel.  Kernel tsolve: one warp per row, Cholesky of the 2^N x 2^N system in fp64
// (unused levels get an identity row -> T = 0, Moore-Penrose, reading R-9); rows whose
// used block is numerically singular fall back to a Jacobi eigen pseudo-inverse.
#include "ganq_internal.cuh"

namespace ganq {
namespace {

constexpr int KC = 128;  // columns k per chunk (32 lanes x float4)
constexpr int JT = 32;   // rows j per H tile
constexpr int WARPS = 8; // rows per CTA

// Sum 16 (or fewer) per-lane bin values across the warp by recursive halving.
// In: v[NB] per lane.  Out: returns the full warp sum of bin `bin_of_lane(lane)`.
template <int NB>
__device__ __forceinline__ float halving_reduce(float (&v)[NB], int lane) {
  // step with offset 16, 8, ... while more than one bin remains
  int nb = NB;
  int off = 16;
#pragma unroll
  for (int step = 0; (1 << step) < NB; ++step) {
    const int half = NB >> (step + 1);
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      // lanes with bit `off` clear keep bins [0, half), others keep [half, 2*half)
      const float send = upper ? v[q] : v[q + half];
      const float keep = upper ? v[q + half] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    off >>= 1;
    nb = half;
  }
  float s = v[0];
  for (; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  (void)nb;
  return s;
}
// Bin held by `lane` after halving_reduce<NB>: bits 4,3,... of lane (msb first) select halves.
template <int NB>
__device__ __forceinline__ int bin_of_lane(int lane) {
  int bin = 0;
  int off = 16;
#pragma unroll
  for (int step = 0; (1 << step) < NB; ++step) {
    const int half = NB >> (step + 1);
    if (lane & off) bin += half;
    off >>= 1;
  }
  return bin;
}

template <int NLEV>
__global__ void __launch_bounds__(WARPS * 32)
tgram_kernel(const float* __restrict__ H32, const float* __restrict__ WH, const uint8_t* __restrict__ Q,
             int64_t m, int64_t n, double* __restrict__ G, double* __restrict__ bvec,
             int* __restrict__ cnt) {
  __shared__ __align__(16) float Hs[JT][KC];
  __shared__ double Cs[WARPS][NLEV][NLEV + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * WARPS + warp;
  const bool live = row < m;
  const uint8_t* q = Q + (live ? row : 0) * n;

  double gacc[NLEV];  // this lane's bin (bin_of_lane) column of C, all a
#pragma unroll
  for (int a = 0; a < NLEV; ++a) gacc[a] = 0.0;
  const int mybin = bin_of_lane<NLEV>(lane);

  const int64_t nchunks = (n + KC - 1) / KC;
  for (int64_t kc = 0; kc < nchunks; ++kc) {
    const int64_t k0 = kc * KC + 4 * lane;
    int bk[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) bk[v] = (live && k0 + v < n) ? (int)q[k0 + v] : -1;
    float acc[NLEV][4];
#pragma unroll
    for (int a = 0; a < NLEV; ++a)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[a][v] = 0.0f;

    for (int64_t j0 = kc * KC; j0 < n; j0 += JT) {  // tiles with some j > k
      __syncthreads();
      for (int idx = threadIdx.x; idx < JT * KC / 4; idx += WARPS * 32) {
        const int jj = idx / (KC / 4), kk = (idx % (KC / 4)) * 4;
        const int64_t j = j0 + jj;
        float4 h;
        float* hp = reinterpret_cast<float*>(&h);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int64_t k = kc * KC + kk + v;
          hp[v] = (j < n && k < n && j > k) ? H32[j * n + k] : 0.0f;
        }
        *reinterpret_cast<float4*>(&Hs[jj][kk]) = h;
      }
      __syncthreads();
      const int64_t jl = j0 + lane;
      const int qj = (live && jl < n) ? (int)q[jl] : -1;
#pragma unroll
      for (int a = 0; a < NLEV; ++a) {
        unsigned msk = __ballot_sync(0xffffffffu, qj == a);
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        while (msk) {
          const int jj = __ffs(msk) - 1;
          msk &= msk - 1;
          const float4 h = *reinterpret_cast<const float4*>(&Hs[jj][4 * lane]);
          s0 += h.x; s1 += h.y; s2 += h.z; s3 += h.w;
        }
        acc[a][0] += s0; acc[a][1] += s1; acc[a][2] += s2; acc[a][3] += s3;
      }
    }
    // scatter acc[a][v] to bins b = bk[v] and reduce over the warp (deterministic)
#pragma unroll
    for (int a = 0; a < NLEV; ++a) {
      float binv[NLEV];
#pragma unroll
      for (int b = 0; b < NLEV; ++b) binv[b] = 0.0f;
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int b = 0; b < NLEV; ++b) binv[b] += (bk[v] == b) ? acc[a][v] : 0.0f;
      const float s = halving_reduce<NLEV>(binv, lane);
      gacc[a] += (double)s;
    }
  }

  // diagonal part D, the right-hand side b and the level counts (lanes over j)
  double dsum[NLEV], rsum[NLEV];
  int c[NLEV];
#pragma unroll
  for (int a = 0; a < NLEV; ++a) { dsum[a] = 0.0; rsum[a] = 0.0; c[a] = 0; }
  if (live) {
    const float* wh = WH + row * n;
    for (int64_t j = lane; j < n; j += 32) {
      const int qj = q[j];
      const double hd = (double)H32[j * n + j];
      const double r = (double)wh[j];
#pragma unroll
      for (int a = 0; a < NLEV; ++a) {
        const bool hit = qj == a;
        dsum[a] += hit ? hd : 0.0;
        rsum[a] += hit ? r : 0.0;
        c[a] += hit ? 1 : 0;
      }
    }
  }
#pragma unroll
  for (int a = 0; a < NLEV; ++a) {
    for (int o = 16; o; o >>= 1) {
      dsum[a] += __shfl_xor_sync(0xffffffffu, dsum[a], o);
      rsum[a] += __shfl_xor_sync(0xffffffffu, rsum[a], o);
      c[a] += __shfl_xor_sync(0xffffffffu, c[a], o);
    }
  }
  // assemble G = C + C^T + D
  const bool writer = (NLEV >= 32) ? true : ((lane & ((32 / NLEV) - 1)) == 0);
  if (writer) {
#pragma unroll
    for (int a = 0; a < NLEV; ++a) Cs[warp][a][mybin] = gacc[a];
  }
  __syncwarp();
  if (live) {
    double* g = G + row * NLEV * NLEV;
    for (int idx = lane; idx < NLEV * NLEV; idx += 32) {
      const int a = idx / NLEV, b = idx % NLEV;
      double v = Cs[warp][a][b] + Cs[warp][b][a];
      if (a == b) {
#pragma unroll
        for (int aa = 0; aa < NLEV; ++aa)
          if (aa == a) v += dsum[aa];
      }
      g[idx] = v;
    }
    if (lane == 0) {
#pragma unroll
      for (int a = 0; a < NLEV; ++a) {
        bvec[row * NLEV + a] = rsum[a];
        cnt[row * NLEV + a] = c[a];
      }
    }
  }
}

// One warp per row; lane l < NLEV holds row l of the (regularised) system.
template <int NLEV>
__global__ void __launch_bounds__(256)
tsolve_kernel(const double* __restrict__ G, const double* __restrict__ bvec, const int* __restrict__ cnt,
              int64_t m, int empty_rule, float* __restrict__ T, int* __restrict__ fallback) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + warp;
  if (row >= m) return;
  const int l = lane < NLEV ? lane : 0;
  const bool used = cnt[row * NLEV + l] > 0;
  double g[NLEV];
  double maxdiag = 0.0;
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double v = G[(row * NLEV + l) * NLEV + c];
    const bool usedc = __shfl_sync(0xffffffffu, used ? 1 : 0, c) != 0;
    g[c] = (used && usedc) ? v : ((c == l && !used) ? 1.0 : 0.0);
  }
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double d = __shfl_sync(0xffffffffu, g[c], c);
    const bool uc = __shfl_sync(0xffffffffu, used ? 1 : 0, c) != 0;
    if (uc && d > maxdiag) maxdiag = d;
  }
  double x = used ? bvec[row * NLEV + l] : 0.0;
  const double tol = (double)NLEV * 2.220446049250313e-16 * maxdiag;
  bool ok = true;
  // Cholesky G = L L^T (lane l keeps row l of L in g[0..l])
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double piv = __shfl_sync(0xffffffffu, g[c], c);
    if (!(piv > tol)) ok = false;
    const double lcc = sqrt(piv > 0.0 ? piv : 1.0);
    double lic = (lane > c) ? g[c] / lcc : (lane == c ? lcc : 0.0);
    if (lane < NLEV) g[c] = lic;
#pragma unroll
    for (int q = c + 1; q < NLEV; ++q) {
      const double lqc = __shfl_sync(0xffffffffu, lic, q);
      if (lane > c && q <= lane) g[q] -= lic * lqc;
    }
  }
  // forward: L y = b
#pragma unroll
  for (int c = 0; c < NLEV; ++c) {
    const double lcc = __shfl_sync(0xffffffffu, g[c], c);
    const double yc = __shfl_sync(0xffffffffu, x, c) / lcc;
    if (lane == c) x = yc;
    else if (lane > c) x -= g[c] * yc;
  }
  // backward: L^T t = y  (L^T row c = column c of L: lane q holds L[q][c] in g[c])
#pragma unroll
  for (int c = NLEV - 1; c >= 0; --c) {
    const double lcc = __shfl_sync(0xffffffffu, g[c], c);
    const double tc = __shfl_sync(0xffffffffu, x, c) / lcc;
    if (lane == c) x = tc;
    // x_r -= L[c][r] * t_c for r < c : lane c holds L[c][r] = g[r]; broadcast per r
#pragma unroll
    for (int r = 0; r < c; ++r) {
      const double lcr = __shfl_sync(0xffffffffu, g[r], c);
      if (lane == r) x -= lcr * tc;
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  if (!ok) {
    if (lane == 0) fallback[row] = 1;
    return;
  }
  if (lane < NLEV) {
    float out = (float)x;
    if (!used) out = (empty_rule == 1) ? T[row * NLEV + lane] : 0.0f;
    T[row * NLEV + lane] = out;
  }
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
ganq_status_t launch_tstep_t(const float* WH, const uint8_t* Q, const float* H32, int64_t m, int64_t n,
                             int empty_rule, float* T, double* G, double* b, int* cnt, int* fb,
                             cudaStream_t st) {
  tgram_kernel<NLEV><<<(unsigned)((m + WARPS - 1) / WARPS), WARPS * 32, 0, st>>>(H32, WH, Q, m, n, G,
                                                                                 b, cnt);
  GANQ_LAUNCH_CHECK("tgram_kernel");
  tsolve_kernel<NLEV><<<(unsigned)((m + 7) / 8), 256, 0, st>>>(G, b, cnt, m, empty_rule, T, fb);
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

ganq_status_t launch_tstep(const float* WH, const uint8_t* Q, const float* H32, int64_t m, int64_t n,
                           int nlev, int empty_rule, float* T, double* G, double* b, int* cnt,
                           int* fb, cudaStream_t st) {
  switch (nlev) {
    case 2: return launch_tstep_t<2>(WH, Q, H32, m, n, empty_rule, T, G, b, cnt, fb, st);
    case 4: return launch_tstep_t<4>(WH, Q, H32, m, n, empty_rule, T, G, b, cnt, fb, st);
    case 8: return launch_tstep_t<8>(WH, Q, H32, m, n, empty_rule, T, G, b, cnt, fb, st);
    case 16: return launch_tstep_t<16>(WH, Q, H32, m, n, empty_rule, T, G, b, cnt, fb, st);
    default:
      set_error(GANQ_ERR_UNSUPPORTED, "tstep: 2^N = %d levels unsupported (N must be 1..4)", nlev);
      return GANQ_ERR_UNSUPPORTED;
  }
}

}  // namespace ganq
