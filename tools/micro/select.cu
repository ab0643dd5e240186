// One warp, the S-step decision chain of sstep_tc (z = w + a; 15 compares against sorted
// thresholds; select tree for t_q; e = w - t_q; feedback FMA into the next column), cycles per
// column.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 select.cu -o select
#include <cstdio>
template <int LO, int HI, typename V, int NLEV>
__device__ __forceinline__ V tree_select(const V (&v)[NLEV], const bool (&p)[NLEV - 1]) {
  if constexpr (LO == HI) {
    return v[LO];
  } else {
    constexpr int MID = (LO + HI) / 2;
    const V lo = tree_select<LO, MID>(v, p);
    const V hi = tree_select<MID + 1, HI>(v, p);
    return p[MID] ? hi : lo;
  }
}
template <int ROWS>
__global__ void chain(float* out, long long* cyc, const float* wsrc, int iters) {
  float v[ROWS][16], th[ROWS][15];
  for (int r = 0; r < ROWS; ++r)
    for (int s = 0; s < 16; ++s) v[r][s] = -0.3f + 0.04f * s + 0.001f * threadIdx.x + 0.01f * r;
  for (int r = 0; r < ROWS; ++r)
    for (int s = 0; s < 15; ++s) th[r][s] = 0.5f * (v[r][s] + v[r][s + 1]);
  float a[ROWS], w[ROWS][8];
  for (int r = 0; r < ROWS; ++r) {
    a[r] = 0.f;
    for (int k = 0; k < 8; ++k) w[r][k] = wsrc[(threadIdx.x + 32 * r + k) & 255];
  }
  const float lc = 0.37f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int cc = 7; cc >= 0; --cc) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const float z = __fadd_rn(w[r][cc], a[r]);
        bool pz[15];
#pragma unroll
        for (int s = 0; s < 15; ++s) pz[s] = z > th[r][s];
        const float tq = tree_select<0, 15>(v[r], pz);
        const float ec = __fsub_rn(w[r][cc], tq);
        a[r] = fmaf(ec, lc, a[r] * 0.5f);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int r = 0; r < ROWS; ++r) s += a[r];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// warp 0: the chain; warp 4 (same SMSP): independent conversions (mode 1) or FFMAs (mode 2)
__global__ void chain_interf(float* out, long long* cyc, const float* wsrc, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  if (warp == 4) {
    int x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    float f0 = 0, f1 = 0, f2 = 0, f3 = 0;
    for (int i = 0; i < iters * 40; ++i) {
      if (mode == 1) {
        f0 += (float)(x0 + i); f1 += (float)(x1 ^ i); f2 += (float)(x2 + 2 * i); f3 += (float)(x3 - i);
      } else {
        f0 = fmaf(f0, 0.999f, 1.f); f1 = fmaf(f1, 0.999f, 1.f); f2 = fmaf(f2, 0.999f, 1.f); f3 = fmaf(f3, 0.999f, 1.f);
      }
    }
    out[threadIdx.x] = f0 + f1 + f2 + f3;
    return;
  }
  if (warp != 0) return;
  float v[16], th[15];
  for (int s = 0; s < 16; ++s) v[s] = -0.3f + 0.04f * s + 0.001f * threadIdx.x;
  for (int s = 0; s < 15; ++s) th[s] = 0.5f * (v[s] + v[s + 1]);
  float a = 0.f, w[8];
  for (int k = 0; k < 8; ++k) w[k] = wsrc[(threadIdx.x + k) & 255];
  const float lc = 0.37f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int cc = 7; cc >= 0; --cc) {
      const float z = __fadd_rn(w[cc], a);
      bool pz[15];
#pragma unroll
      for (int s = 0; s < 15; ++s) pz[s] = z > th[s];
      const float tq = tree_select<0, 15>(v, pz);
      const float ec = __fsub_rn(w[cc], tq);
      a = fmaf(ec, lc, a * 0.5f);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  float *out, *w;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMallocManaged(&w, 256 * 4);
  for (int i = 0; i < 256; ++i) w[i] = -0.3f + 0.6f * ((i * 37) % 256) / 256.f;
  cudaMallocManaged(&cyc, 64);
  const int iters = 2048;
  chain<1><<<1, 32>>>(out, cyc, w, iters);
  cudaDeviceSynchronize();
  chain<1><<<1, 32>>>(out, cyc, w, iters);
  cudaDeviceSynchronize();
  printf("1 row/lane: %.1f cycles per column\n", (double)cyc[0] / (iters * 8));
  chain<2><<<1, 32>>>(out, cyc, w, iters);
  cudaDeviceSynchronize();
  chain<2><<<1, 32>>>(out, cyc, w, iters);
  cudaDeviceSynchronize();
  printf("2 rows/lane: %.1f cycles per column (both rows)\n", (double)cyc[0] / (iters * 8));
  for (int mode = 1; mode <= 2; ++mode) {
    chain_interf<<<1, 160>>>(out, cyc, w, iters, mode);
    cudaDeviceSynchronize();
    chain_interf<<<1, 160>>>(out, cyc, w, iters, mode);
    cudaDeviceSynchronize();
    printf("with a co-resident %s warp on the same SMSP: %.1f cycles per column\n",
           mode == 1 ? "I2F+FADD" : "FFMA", (double)cyc[0] / (iters * 8));
  }
  return 0;
}
