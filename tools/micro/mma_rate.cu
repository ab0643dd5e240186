// tcgen05.mma kind::i8 issue rate, A from shared memory (ss) vs from TMEM (ts), M = 128,
// N = 64 / 128 / 256, K = 32 per instruction; one CTA per SM, one thread issues R MMAs
// back to back into one accumulator, then commits and waits.   nvcc -arch=sm_100a ...
#include <cstdio>
#include "../../paper_2501_12956_b200/csrc/ganq_internal.cuh"
using namespace ganq;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_rate(long long* cyc, int R) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* a = sm;            // 128 x 64 B (SW64)
  uint8_t* b = sm + 8192;     // N x 64 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (8192 + N * 64) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01010101u * (i & 1), 0, 0x02020202u, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_u8s8(128, N);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        if (TS) mma_i8_ts(tm, tm + 384 + kk * 8, umma_desc_sw64(sb + kk * 32), idesc, (r | kk) ? 1u : 0u);
        else mma_i8(tm, umma_desc_sw64(sa + kk * 32), umma_desc_sw64(sb + kk * 32), idesc, (r | kk) ? 1u : 0u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

// the tgram pattern: per stage 3 digit accumulators x 2 K-steps, A from TMEM, then (MODE >= 1)
// a commit per stage and (MODE >= 2) a wait on an already-completed mbarrier per stage
template <int MODE>
__global__ void __launch_bounds__(128, 1) k_pattern(long long* cyc, int R) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* b = sm;  // 3 digit tiles of 128 x 64 B
  __shared__ uint64_t bar, ready, fullb;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 3 * 8192 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01010101u, 0, 2, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&ready, 1); mbar_init(&fullb, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    mbar_arrive(&ready);  // phase 0 complete: waits on parity 0 return at once
    constexpr uint32_t idesc = umma_idesc_u8s8(128, 128);
    const uint32_t sb = smem_u32(b);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      if (MODE == 2) mbar_wait(&ready, 0);
      if (MODE == 3) {  // non-blocking test_wait poll instead of try_wait
        uint32_t ok = 0;
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&ready)), "r"(0) : "memory");
        } while (!ok);
      }
      tc_fence_after();
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          mma_i8_ts(tm + l * 128, tm + 384 + (r % 6) * 16 + kk * 8, umma_desc_sw64(sb + l * 8192 + kk * 32),
                    idesc, (r | kk) ? 1u : 0u);
      if (MODE >= 1) mma_commit(&fullb);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}
// the tgram pattern under concurrent traffic: warps 1-4 store to TMEM (tcgen05.st, the
// producers' one-hot ring) and/or warps 5-8 write shared memory (like TMA fills / the epilogue)
template <bool TST, bool SST>
__global__ void __launch_bounds__(288, 1) k_contend(long long* cyc, int R) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* b = sm;  // 3 digit tiles of 128 x 128 B (SW128)
  uint8_t* scratch = sm + 3 * 16384;
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 3 * 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01010101u, 0, 2, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); stop = 0; fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_u8s8(128, 128);
    const uint32_t sb = smem_u32(b);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8_ts(tm + l * 128, tm + 384 + (r % 3) * 32 + kk * 8, umma_desc_sw128(sb + l * 16384 + kk * 32, 16, 1024),
                    idesc, (r | kk) ? 1u : 0u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = t1 - t0;
    stop = 1;
  } else if (TST && warp >= 1 && warp <= 4) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = i;
    const uint32_t ta = tm + ((uint32_t)((warp & 3) * 32) << 16) + 480;
    while (!stop) { tmem_st16(ta, v); tmem_st16(ta + 16, v); tmem_st_wait(); }
  } else if (SST && warp >= 5) {
    uint4* sp = reinterpret_cast<uint4*>(scratch) + (threadIdx.x - 160);
    uint4 z = make_uint4(threadIdx.x, 1, 2, 3);
    while (!stop) {
#pragma unroll 8
      for (int i = 0; i < 64; ++i) sp[(i * 128) % 4096] = z;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}
template <bool TST, bool SST>
void runc(long long* cyc) {
  const int R = 1000, smem = 3 * 16384 + 65536 + 1024;
  cudaFuncSetAttribute(k_contend<TST, SST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_contend<TST, SST><<<148, 288, smem>>>(cyc, 50);
  k_contend<TST, SST><<<148, 288, smem>>>(cyc, R);
  cudaError_t e = cudaDeviceSynchronize();
  printf("12-MMA stages, tcgen05.st traffic %d, smem-write traffic %d: %.1f cycles per MMA  %s\n", (int)TST, (int)SST,
         (double)cyc[0] / (12.0 * R), cudaGetErrorString(e));
}

template <int MODE>
void runp(long long* cyc) {
  const int R = 2000, smem = 3 * 8192 + 1024;
  cudaFuncSetAttribute(k_pattern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_pattern<MODE><<<148, 128, smem>>>(cyc, 100);
  k_pattern<MODE><<<148, 128, smem>>>(cyc, R);
  cudaError_t e = cudaDeviceSynchronize();
  printf("tgram pattern mode %d: %.1f cycles per MMA  %s\n", MODE, (double)cyc[0] / (6.0 * R), cudaGetErrorString(e));
}

template <int N, bool TS>
void run(long long* cyc) {
  const int R = 4000, smem = 8192 + N * 64 + 1024;
  cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_rate<N, TS><<<148, 128, smem>>>(cyc, 100);
  k_rate<N, TS><<<148, 128, smem>>>(cyc, R);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s N=%3d: %.1f cycles per MMA (floor N/2 = %d)  %s\n", TS ? "ts" : "ss", N, (double)cyc[0] / (2.0 * R), N / 2,
         cudaGetErrorString(e));
}
int main() {
  long long* cyc;
  cudaMallocManaged(&cyc, 64);
  run<64, false>(cyc); run<128, false>(cyc); run<256, false>(cyc);
  run<64, true>(cyc); run<128, true>(cyc); run<256, true>(cyc);
  runp<0>(cyc); runp<1>(cyc); runp<2>(cyc); runp<3>(cyc);
  runc<false, false>(cyc); runc<true, false>(cyc); runc<false, true>(cyc); runc<true, true>(cyc);
  return 0;
}
