// ganq_internal.cuh -- internal helpers for the sm_100a GANQ kernels.
// Not part of the public ABI (include/ganq.h).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ganq.h"

namespace ganq {

// ---------------------------------------------------------------- error state
void set_error(ganq_status_t st, const char* fmt, ...);
void set_error_index(int64_t idx);
// validate.cu: GANQ_VALIDATE=1 scans inputs for Inf / NaN (synchronises; INVALID_ARG on a hit)
bool validate_enabled();
ganq_status_t validate_finite_f32(const float* x, int64_t rows, int64_t cols, const char* what, cudaStream_t st);
ganq_status_t validate_finite_f64(const double* x, int64_t rows, int64_t cols, const char* what, cudaStream_t st);
ganq_status_t validate_finite_bf16(const uint16_t* x, int64_t rows, int64_t cols, const char* what,
                                   cudaStream_t st);
ganq_status_t cuda_fail(cudaError_t e, const char* where);

#define GANQ_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::ganq::cuda_fail(_e, #expr); \
  } while (0)

void count_launch();

#define GANQ_LAUNCH_CHECK(where)                                         \
  do {                                                                   \
    ::ganq::count_launch();                                              \
    cudaError_t _e = cudaGetLastError();                                 \
    if (_e != cudaSuccess) return ::ganq::cuda_fail(_e, where);          \
  } while (0)

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- launchers (internal)
// hessian.cu
int hessian_tiles(int64_t n);
int64_t hessian_superchunks(int64_t p);
size_t hessian_fixed_bytes(int64_t n);
size_t hessian_partials_bytes(int64_t p, int64_t n);
ganq_status_t check_hessian_args(const uint16_t* X, int64_t p, int64_t n);
// super-chunk partials (fp32) of X X^T and the channel exponent bounds E (assigned)
ganq_status_t launch_hessian_partials(const uint16_t* X, int64_t p, int64_t n, float* Psc, int32_t* E,
                                      cudaStream_t st);
ganq_status_t launch_hessian_fixed(const float* Psc, int64_t p, int64_t n, const int32_t* E, long long* Hfix,
                                   int accumulate, cudaStream_t st);
// H from Hfix, or (Psc != nullptr) straight from the partials of p tokens
ganq_status_t launch_hessian_finalize(const long long* Hfix, const float* Psc, int64_t p, const int32_t* E, int64_t n,
                                      double* H, int accumulate, cudaStream_t st);
// cholesky.cu
ganq_status_t launch_precondition(const double* H, int64_t n, int policy, double lambda, double tau,
                                  double* A, double* delta, double* d_mean, cudaStream_t st);
// d_ticket: a device int that is 0 on entry (the panel kernel's completion counter; left 0)
ganq_status_t launch_cholesky(double* A, int64_t n, int* d_status, int* d_ticket, cudaStream_t st);
ganq_status_t launch_derive_operands(const double* L, const double* H, int64_t n, float* Lhat,
                                     float* H32, cudaStream_t st);
// tstep.cu
ganq_status_t launch_kmeans_codebook(const float* W, int64_t m, int64_t n, int nlev, int iters, float* T,
                                     cudaStream_t st);
ganq_status_t launch_init_codebook(const float* W, int64_t m, int64_t n, int nlev, float* T,
                                   cudaStream_t st);
// the T-update after the normal matrices (launch_tgram_tc): right-hand sides and the solves
ganq_status_t launch_hdiag(const double* H, int64_t n, double* hdiag, cudaStream_t st);  // H_jj, once per layer
ganq_status_t launch_tsolve(const double* hdiag, const float* WH, const uint8_t* Q, int64_t m, int64_t n, int nlev,
                            int empty_rule, float* T, double* G, double* Dv, double* b, int* cnt, int* fallback,
                            cudaStream_t st);
// lut.cu (NEXT-1)
ganq_status_t launch_pack_codes(const uint8_t* Q, int64_t m, int64_t n, int N, uint8_t* P, cudaStream_t st);
ganq_status_t launch_codebook_f16(const float* T, int64_t total, uint16_t* T16, cudaStream_t st);
ganq_status_t launch_lut_gemm(const uint8_t* P, const uint16_t* T16, const uint16_t* X, int64_t m, int64_t n,
                              int64_t p, int N, float* Y, cudaStream_t st);
// outlier.cu (NEXT-2)
void outlier_indices(int64_t n, double r, int64_t* up, int64_t* lo);
ganq_status_t launch_outlier_split(const float* W, int64_t m, int64_t n, double r, float* Wd, float* c_lo,
                                   float* c_hi, int64_t* off, cudaStream_t st);
ganq_status_t launch_outlier_csr(const float* W, int64_t m, int64_t n, const float* c_lo, const float* c_hi,
                                 const int64_t* off, int32_t* col, float* val, cudaStream_t st);
ganq_status_t launch_sparse_gemm_add(const int64_t* off, const int32_t* col, const float* val, int64_t m, int64_t n,
                                     const uint16_t* X, int64_t p, float* Y, cudaStream_t st);
// tgram_tc.cu
int64_t tq_pitch(int64_t n);
int tgram_splits(int64_t m, int nlev);  // CTAs per row group of the normal-matrix kernel (1..4)
ganq_status_t launch_tq_prep(const double* H, int64_t n, int8_t* Hq, double* scale, cudaStream_t st);
ganq_status_t launch_tgram_tc(const int8_t* Hq, const double* scale, const uint8_t* Q, int64_t m,
                              int64_t n, int nlev, double* Cg, cudaStream_t st);
// sstep_tc.cu
int64_t ss_pitch(int64_t n);   // fp32 Lhat row pitch (multiple of 4)
int64_t ssq_pitch(int64_t n);  // int8 digit-plane row pitch (multiple of 64); n_blocks = ssq_pitch / 64
int64_t ss_panels(int64_t n);  // 128-column panels of the S-step
// Lhat (fp32, in-panel feedback) and the 24-bit digits of LhatT with their scales per (source
// panel, column) tLp[ss_panels(n)][n] (bmax: scratch of ssq_pitch(n) / 64 * n floats)
ganq_status_t launch_lhat_prep(const double* L, int64_t n, float* Lhat, int8_t* LTq, float* tLp, float* bmax,
                               cudaStream_t st);
// sEp: the residual digits' scales per (source panel, row), ss_panels(n) x ceil32(m) floats
ganq_status_t launch_sstep_tc(const float* W, const float* Lhat, const int8_t* LTq, const float* tLp,
                              const float* T, int64_t m, int64_t n, int nlev, uint8_t* Q, int8_t* Eq,
                              float* sEp, cudaStream_t st);
// gemm_tc.cu
int64_t gemm_pitch(int64_t K);
ganq_status_t launch_split_tf32(const float* X, int64_t rows, int64_t K, float* hi, float* lo,
                                cudaStream_t st);
ganq_status_t launch_gemm_tf32x3(const float* Ahi, const float* Alo, const float* Bhi, const float* Blo,
                                 int64_t M, int64_t N, int64_t K, float* C, cudaStream_t st);
// gemm.cu
ganq_status_t launch_residual(const float* W, const uint8_t* Q, const float* T, int64_t m, int64_t n,
                              int nlev, float* E, cudaStream_t st);
ganq_status_t launch_rowdot(const float* E, const float* EH, int64_t m, int64_t n, double* per_row,
                            cudaStream_t st);
ganq_status_t launch_sum(const double* x, int64_t m, double* out, cudaStream_t st);

// ---------------------------------------------------------------- device PTX helpers
#if defined(__CUDACC__)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA 2D tile load global -> shared, completion signalled on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA 3D tile load (coordinates innermost first); out-of-range boxes are zero-filled.
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* smem_dst, const void* tmap, uint64_t* bar, int c0,
                                               int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
// TMA 2D tile load multicast to the CTAs of `mask` in the cluster (same smem offsets and
// mbarrier offset in every destination CTA).
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const void* tmap, uint64_t* bar, int c0,
                                               int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// tcgen05 (5th-gen tensor core) wrappers.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc]; kind::f16 (bf16 inputs here), fp32 accumulate.
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Arrive on the mbarrier at the same offset in every CTA of `mask` once the MMAs complete.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// 32 lanes x 32 bit, 8 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(taddr));
}
// 32 lanes x 32 bit, 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// D[tmem] (+)= A * B with signed int8 operands and exact int32 accumulation (kind::i8).
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One pipeline stage of the one-hot T-update contraction, issued by ONE elected lane of a
// converged warp in a single asm block: for digit l = 0..2 and k-step kk = 0..3,
//   D[d_tmem + 128 l] (+)= A[a_tmem + 8 kk] * B[bdesc + (l * DIG + 32 kk) bytes]
// (kind::i8, A from TMEM), then the MMAs' completion arrives on `bar` in every CTA of `mask`.
// `first` != 0 overwrites each accumulator with its kk = 0 product.  Issuing the twelve MMAs
// under one elect.sync (descriptors advanced by immediates) keeps the issuer's instruction
// chain per MMA shorter than the 64-cycle MMA itself.  DIG = the byte stride of the digit tiles
// (16 KB single CTA, 8 KB per CTA of a pair); CG = cta_group.
#define GANQ_STAGE12(NAME, CG, D1, D2)                                                                    \
  __device__ __forceinline__ void NAME(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, \
                                       uint32_t first, uint64_t* bar, uint16_t mask) {                   \
    asm volatile(                                                                                        \
        "{\n\t"                                                                                          \
        ".reg .pred e, acc;\n\t"                                                                         \
        ".reg .b32 d1, d2, a1, a2, a3;\n\t"                                                              \
        ".reg .b64 b;\n\t"                                                                               \
        "elect.sync _|e, 0xffffffff;\n\t"                                                                \
        "setp.eq.b32 acc, %4, 0;\n\t"                                                                    \
        "add.u32 d1, %0, 128;\n\t"                                                                       \
        "add.u32 d2, %0, 256;\n\t"                                                                       \
        "add.u32 a1, %1, 8;\n\t"                                                                         \
        "add.u32 a2, %1, 16;\n\t"                                                                        \
        "add.u32 a3, %1, 24;\n\t"                                                                        \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [%0], [%1], %2, %3, acc;\n\t"                         \
        "add.s64 b, %2, " D1 ";\n\t"                                                                     \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d1], [%1], b, %3, acc;\n\t"                          \
        "add.s64 b, %2, " D2 ";\n\t"                                                                     \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d2], [%1], b, %3, acc;\n\t"                          \
        "add.s64 b, %2, 2;\n\t"                                                                          \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [%0], [a1], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, " D1 "+2;\n\t"                                                                   \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d1], [a1], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, " D2 "+2;\n\t"                                                                   \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d2], [a1], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, 4;\n\t"                                                                          \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [%0], [a2], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, " D1 "+4;\n\t"                                                                   \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d1], [a2], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, " D2 "+4;\n\t"                                                                   \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d2], [a2], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, 6;\n\t"                                                                          \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [%0], [a3], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, " D1 "+6;\n\t"                                                                   \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d1], [a3], b, %3, 1;\n\t"                            \
        "add.s64 b, %2, " D2 "+6;\n\t"                                                                   \
        "@e tcgen05.mma.cta_group::" CG ".kind::i8 [d2], [a3], b, %3, 1;\n\t"                            \
        "@e tcgen05.commit.cta_group::" CG                                                               \
        ".mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %6;\n\t"                    \
        "}\n" ::"r"(d_tmem),                                                                             \
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(first), "r"(smem_u32(bar)), "h"(mask)                   \
        : "memory");                                                                                     \
  }
// descriptor units are 16 bytes: 16 KB = 1024
GANQ_STAGE12(mma_i8_ts_stage12_mc, "1", "1024", "2048")
#undef GANQ_STAGE12
// CTA-pair (cta_group::2) variants: issued by the leader CTA; A rows 0-127 / 128-255 and the
// two N halves of B live at the same TMEM / shared offsets of the two CTAs.
__device__ __forceinline__ void mma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// TMA 2D load into this CTA's shared memory, completion counted on the pair leader's mbarrier
// (same offset; the peer bit of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* tmap, uint64_t* bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
// mbarrier arrive on the copy of `bar` in CTA `rank` of the cluster.  Default semantics
// (release at CTA scope, as CUTLASS's ClusterBarrier::arrive): enough to hand TMEM back to the
// pair's MMA issuer after tcgen05.wait::ld + tcgen05.fence::before_thread_sync, and it does not
// drain this warp's outstanding global stores (a .release.cluster arrive compiles to a
// MEMBAR.ALL.GPU).
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t"
      ".reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread, registers -> TMEM.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// signal a named barrier without waiting (producer side of a bar.sync by other warps)
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory matrix descriptor (sm_100 "version 1"), 128B swizzle.
//   bits [0,14)  start address >> 4      bits [16,30) leading byte offset >> 4
//   bits [32,46) stride byte offset >> 4 bits [46,48) version = 1
//   bits [49,52) base offset = 0         bit  52      lbo mode = 0
//   bits [61,64) layout: 2 = SWIZZLE_128B
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor for kind::f16 / kind::tf32 with fp32 accumulation.
//   [4,6) c_format (1 = F32)   [7,10) a_format   [10,13) b_format (BF16 = 1, TF32 = 2)
//   [15] a_major (1 = MN)      [16] b_major      [17,23) N >> 3     [24,29) M >> 4
__host__ __device__ constexpr uint32_t umma_idesc(uint32_t ab_format, uint32_t a_mn_major,
                                                  uint32_t b_mn_major, uint32_t M, uint32_t N) {
  return (1u << 4) | (ab_format << 7) | (ab_format << 10) | (a_mn_major << 15) |
         (b_mn_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
// kind::i8: signed int8 A and B (format 1), S32 accumulator (c_format 2), K-major operands.
// K-major SWIZZLE_64B UMMA smem descriptor: 64-byte rows, 8-row atoms of 512 B (SBO),
// layout type 4 (the TMA SWIZZLE_64B image of a box with a 64-byte inner extent).
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t umma_idesc_s8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
// kind::i8 with an unsigned (u8) A operand and a signed (s8) B operand, s32 accumulate
__host__ __device__ constexpr uint32_t umma_idesc_u8s8(uint32_t M, uint32_t N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
#endif

}  // namespace ganq
