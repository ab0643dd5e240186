/*
 * ganq.h -- C ABI of the B200 (sm_100a) GANQ layer-quantization solver.
 *
 * GANQ (arxiv 2501.12956): GPU-adaptive layer-wise LUT-based non-uniform
 * quantization.  For one linear layer W (m x n) and calibration activations X
 * (n x p) it minimises the layer output error
 *       min_{Q,T} || W X - W~ X ||_F^2 ,  W~_ij = T_{i, Q_ij}          Eq. (1)
 * by Algorithm 1: H = X X^T, L = Cholesky(H'), then K times
 *   S-update: row-parallel back-substitution, column j = n-1 .. 0,
 *             Q_ij = argmin_s | W_ij + (1/L_jj) sum_{u>j} r_u L_uj - T_is |   Eq. (22)
 *   T-update: T_i = W_i H S_i^T (S_i H S_i^T)^dagger                           Eq. (6),
 * P:n refers to /root/reference/PAPER.md line n; R-x to the readings listed
 * in DESIGN.md ("Readings of the paper").
 *
 * Conventions (all entry points):
 *  - Every array pointer is a DEVICE pointer (cudaMalloc / torch CUDA memory)
 *    unless the argument says HOST.  All matrices are row-major, dense,
 *    contiguous.  The caller owns every buffer; the library never allocates or
 *    frees user memory (internal scratch lives in the caller's workspace; ganq_hessian alone
 *    draws its scratch from the stream-ordered pool, ganq_hessian_ws takes the caller's).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Work is enqueued on it.  Calls that return a HOST value or
 *    detect a data-dependent error (non-positive-definite factor) synchronise
 *    the stream before returning; this is stated per call.
 *  - Return value: GANQ_OK or an error code; ganq_last_error() gives a
 *    thread-local message.  On error, outputs are unspecified.
 *  - Rows are independent (Eq. 2): a row shard is W + r0*n with
 *    m = m_local; multi-GPU needs no further entry point.
 *  - Non-finite inputs (Inf / NaN in X, W or H) are undefined behaviour.  With the
 *    environment variable GANQ_VALIDATE=1, ganq_hessian and ganq_quantize_layer scan
 *    their inputs first, synchronise, and return GANQ_ERR_INVALID_ARG naming the first
 *    non-finite element (ganq_last_error_index() = its flat index).
 */
#ifndef GANQ_H_
#define GANQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GANQ_OK = 0,
  GANQ_ERR_INVALID_ARG = 1, /* a size/bit-width/iteration/policy argument is out of range   */
  GANQ_ERR_NOT_PD = 2,      /* Cholesky met a non-positive pivot; index in ganq_last_error_index() */
  GANQ_ERR_CUDA = 3,        /* a CUDA runtime/driver call or kernel launch failed            */
  GANQ_ERR_WORKSPACE = 4,   /* workspace NULL or smaller than ganq_workspace_size()          */
  GANQ_ERR_UNSUPPORTED = 5  /* valid but unsupported shape (see the call's notes)            */
} ganq_status_t;

/* Preconditioning of H before the Cholesky factorisation (reading R-3). */
typedef enum {
  GANQ_PRECOND_ADAPTIVE = 0,     /* App. A, Eqs. 23-24: H + Diag(delta),
                                    delta_i = max(sum_j|H_ij| - 2 H_ii, 1e-8) + tau*mean(diag H) */
  GANQ_PRECOND_FIXED_LAMBDA = 1, /* Remark 1: H + lambda I, lambda > 0 */
  GANQ_PRECOND_NONE = 2          /* Algorithm 1 literally: Cholesky(H) */
} ganq_precond_t;

typedef struct {
  int32_t precond;          /* ganq_precond_t; default GANQ_PRECOND_ADAPTIVE                       */
  int32_t empty_level_rule; /* 0 = Moore-Penrose (unused level -> 0, default);
                               1 = keep the previous value (reading R-9 option)                   */
  double lambda;            /* used iff precond == FIXED_LAMBDA; must be > 0                       */
  double tau;               /* ADAPTIVE jitter factor (reading R-3); default 1e-7                  */
  const float* T0;          /* nullable DEVICE m x 2^N initial codebook; NULL -> fp32 min-max grid
                               (reading R-6)                                                        */
  double* obj_trace;        /* nullable HOST array [iters]: Eq. (1) after every T-update; when set
                               the call synchronises the stream once per iteration                 */
} ganq_opts_t;

/* Fill *opts with the defaults listed above.  Never fails. */
void ganq_default_opts(ganq_opts_t* opts);

/*
 * H = X X^T  (Algorithm 1, "Compute H = XX^T"; X is n x p).
 *   X     : DEVICE, p x n bf16 (passed as uint16 bit patterns), TOKEN-major -- row t is the
 *           activation x_t of one calibration token (so X here is the paper's X^T); 16-byte aligned.
 *   p, n  : tokens in [1, 2^31), channels >= 1; n % 8 == 0 is required (TMA row pitch; else
 *           GANQ_ERR_UNSUPPORTED).
 *   H     : DEVICE, n x n fp64, the FULL symmetric matrix is written.
 *   accumulate : 0 -> H = X X^T;  1 -> H += X X^T, added in fp64 (streamed calibration batches).
 * Arithmetic (reading R-12): the tokens are cut into super-chunks of GANQ_HESSIAN_SUPERCHUNK
 * counted from token 0, each accumulated by the tensor cores (tcgen05, CTA pairs, fp32) in
 * chains of 256 tokens folded into a round-to-nearest fp32 sum (the super-chunk's partial);
 * every partial is rounded onto the integer grid 2^(E_i + E_j - 46) (E_c = ceil(e/2) + 1 for
 * max over the super-chunks of the diagonal partial P[c][c] = m 2^e, m in [0.5, 1)) and the
 * super-chunks are added EXACTLY in int64; H = that integer x grid (one rounding to fp64).  The
 * result does not depend on how the super-chunks are grouped: token shards reduced through
 * ganq_hessian_partials / _fixed + integer all-reduces give bitwise the same H as one call.
 * ganq_hessian takes its scratch (ganq_hessian_workspace_size(p, n) bytes) from the device's
 * stream-ordered pool (cudaMallocAsync / cudaFreeAsync on `stream`); ganq_hessian_ws uses the
 * caller's.  Asynchronous on `stream`.
 */
#define GANQ_HESSIAN_SUPERCHUNK 32768
ganq_status_t ganq_hessian(const uint16_t* X, int64_t p, int64_t n, double* H, int accumulate,
                           void* stream);
size_t ganq_hessian_workspace_size(int64_t p, int64_t n);
ganq_status_t ganq_hessian_ws(const uint16_t* X, int64_t p, int64_t n, double* H, int accumulate, void* workspace,
                              size_t workspace_bytes, void* stream);

/*
 * The same computation in its three steps, for token shards (one rank per shard; multi-GPU):
 *   ganq_hessian_partials: partials (DEVICE fp32, ganq_hessian_partials_size(p, n) bytes) = one
 *     fp32 sum per super-chunk of X (X's first token starts a super-chunk: shard boundaries must
 *     be multiples of GANQ_HESSIAN_SUPERCHUNK), and E (DEVICE int32 [n]) = the grid exponents
 *     of its super-chunks' diagonals (above).  Reduce E with MAX over the shards: every shard
 *     must then use the same, global E.
 *   ganq_hessian_fixed: Hfix (DEVICE int64, ganq_hessian_fixed_size(n) bytes, tile-major lower
 *     triangle) = (accumulate ? Hfix + : ) the partials of p tokens rounded onto the grid of E and
 *     summed exactly.  Hfix of several shards adds exactly (int64 SUM all-reduce, any order).
 *   ganq_hessian_finalize: H (DEVICE fp64 n x n, full symmetric) = (accumulate ? H + : ) Hfix x grid.
 * An E below the MAX over all shards' E can make the integers overflow (undefined).  All asynchronous.
 */
size_t ganq_hessian_partials_size(int64_t p, int64_t n);
size_t ganq_hessian_fixed_size(int64_t n);
ganq_status_t ganq_hessian_partials(const uint16_t* X, int64_t p, int64_t n, float* partials, int32_t* E,
                                    void* stream);
ganq_status_t ganq_hessian_fixed(const float* partials, int64_t p, int64_t n, const int32_t* E, int64_t* Hfix,
                                 int accumulate, void* stream);
ganq_status_t ganq_hessian_finalize(const int64_t* Hfix, const int32_t* E, int64_t n, double* H, int accumulate,
                                    void* stream);

/*
 * Bytes of DEVICE workspace ganq_quantize_layer needs for (m, n, n_bits).
 * Returns 0 for invalid arguments.  Independent of iters and options.
 */
size_t ganq_workspace_size(int64_t m, int64_t n, int n_bits);

/*
 * Algorithm 1 for one layer, given H.
 *   W      : DEVICE, m x n fp32 weights (row i = output channel i).
 *   H      : DEVICE, n x n fp64 symmetric X X^T (only read; the T-update uses raw H, reading R-4;
 *            the S-update uses L = Cholesky(precondition(H))).
 *   n_bits : N in [1, 8] is valid; this build solves N <= 4 (2^N <= 16 levels, the paper's 3-
 *            and 4-bit settings) and returns GANQ_ERR_UNSUPPORTED for N = 5..8.
 *            iters: K >= 1 full (S, T) pairs (reading R-5).
 *   opts   : nullable -> ganq_default_opts().
 *   Q      : DEVICE, m x n uint8 output, one code per byte, values < 2^N (Q^K).
 *   T      : DEVICE, m x 2^N fp32 output codebook T^K.
 *   workspace / workspace_bytes : DEVICE scratch of at least ganq_workspace_size(m, n, n_bits).
 * Errors: INVALID_ARG (m, n < 1; n_bits outside [1,8]; iters < 1; unknown policy;
 * lambda <= 0 under FIXED_LAMBDA), WORKSPACE, NOT_PD (index of the failing pivot; possible only
 * for NONE or a tiny lambda), CUDA.
 * Synchronisation: the stream is synchronised once after the factorisation (to report NOT_PD)
 * and once per iteration if opts->obj_trace is set; otherwise the K iterations are enqueued
 * asynchronously.
 */
ganq_status_t ganq_quantize_layer(const float* W, int64_t m, int64_t n, const double* H,
                                  int n_bits, int iters, const ganq_opts_t* opts, uint8_t* Q,
                                  float* T, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Layer objective Eq. (1), evaluated as sum_i e_i H e_i^T with e_i = W_i - W~_i
 * (Eq. 8) on raw H.
 *   out     : HOST double (required).   per_row : nullable DEVICE fp64 [m].
 *   workspace: DEVICE scratch of >= ganq_objective_workspace_size(m, n) bytes.
 * Synchronises the stream (host result).
 */
size_t ganq_objective_workspace_size(int64_t m, int64_t n);
ganq_status_t ganq_objective(const float* W, const uint8_t* Q, const float* T, const double* H,
                             int64_t m, int64_t n, int n_bits, double* out, double* per_row,
                             void* workspace, size_t workspace_bytes, void* stream);

/*
 * T-update alone (Eq. 6; Algorithm 1 "batch update") for given codes:
 *   T_i = W_i H S_i^T (S_i H S_i^T)^dagger, raw H, unused levels per empty_level_rule
 *   (Tprev, DEVICE m x 2^N, read only when empty_level_rule == 1; may alias T).
 * Uses ganq_workspace_size(m, n, n_bits) bytes of workspace.  Asynchronous.
 */
ganq_status_t ganq_tstep(const float* W, const uint8_t* Q, const double* H, int64_t m, int64_t n,
                         int n_bits, int empty_level_rule, const float* Tprev, float* T,
                         void* workspace, size_t workspace_bytes, void* stream);

/*
 * Preconditioned Cholesky factor alone (App. A / Remark 1 / Eq. 9):
 *   L (DEVICE n x n fp64, lower triangle written, strict upper set to 0) = Cholesky(H'),
 *   delta (nullable DEVICE fp64 [n]) = the diagonal offset added.
 * Uses ganq_workspace_size(1, n, 1) bytes of workspace.  Synchronises (reports NOT_PD).
 */
ganq_status_t ganq_factor(const double* H, int64_t n, const ganq_opts_t* opts, double* L,
                          double* delta, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Instrumentation (for bench.py; off by default, no effect on results).
 * ganq_profile_enable(1) resets and starts per-stage timing: every stage of every later
 * call on this thread is bracketed by CUDA events recorded on the call's stream.
 * ganq_profile_read() synchronises those events and fills ms[i] (summed device time) and
 * launches[i] (kernel launches) for stage i < GANQ_PROFILE_STAGES; returns the stage count.
 * ganq_launch_count() is the total number of kernels this library launched (process-wide).
 */
#define GANQ_PROFILE_STAGES 13
int ganq_profile_enable(int on);
int ganq_profile_read(double* ms, int64_t* launches, int max_stages);
const char* ganq_profile_stage_name(int stage);
int64_t ganq_launch_count(void);

/* Thread-local message of the last error on this thread ("" if none). */
const char* ganq_last_error(void);
/* Failing pivot index for GANQ_ERR_NOT_PD, else -1. */
int64_t ganq_last_error_index(void);
/* Library version string. */
/*
 * ---------------------------------------------------------------- NEXT-1: deployment side
 * LUT-based mixed-precision GEMM, Fig. 1a right: W~_ij = t_{i, Q_ij} is never
 * formed; the kernel gathers codebook entries by the packed codes.  Storage as in Table 1
 * (P:87-99): codes N bits each, codebook fp16 (2 * 2^N bytes per row).
 *
 * Packed layout: row i is a little-endian bitstream, code k in bits [k N, (k+1) N), padded to
 * whole bytes: ganq_packed_row_bytes(n, N) = ceil(n N / 8) bytes per row, rows contiguous.
 * fp16 values are passed as their IEEE binary16 bit patterns (uint16_t).
 */
int64_t ganq_packed_row_bytes(int64_t n, int n_bits);

/* Q (m x n codes, < 2^n_bits; larger values are undefined -- only their low n_bits bits are
 * stored) -> packed (m x ganq_packed_row_bytes(n, n_bits)).  Async on `stream`.
 * INVALID_ARG: m, n < 1, n_bits not in [1, 8], null pointers. */
ganq_status_t ganq_pack_codes(const uint8_t* Q, int64_t m, int64_t n, int n_bits, uint8_t* packed,
                              void* stream);

/* T (m x 2^n_bits fp32) -> T16 (m x 2^n_bits fp16, round to nearest even).  Async. */
ganq_status_t ganq_codebook_f16(const float* T, int64_t m, int n_bits, uint16_t* T16, void* stream);

/* Y (p x m, fp32) = X W~^T with X (p x n, fp16, token-major), W~_ij = T16[i][Q_ij] decoded
 * from `packed`.  Each output is accumulated in fp32 in a fixed order (a lane's codes in
 * ascending j, then a fixed butterfly over the 32 lanes of a warp), so results are
 * reproducible run to run.  Intended for decode (p small); p is processed in blocks of 8.
 * Async.  INVALID_ARG: m, n, p < 1, n_bits not in [1, 8], null pointers. */
ganq_status_t ganq_lut_gemm(const uint8_t* packed, const uint16_t* T16, const uint16_t* X, int64_t m,
                            int64_t n, int64_t p, int n_bits, float* Y, void* stream);

/*
 * ---------------------------------------------------------------- NEXT-2: GANQ* outlier split
 * Algorithm 2 (Appendix B; §3.3).  Per row, with p = 1 - 0.5 r, the
 * cutoffs are the row's ascending order statistics at 0-based indices floor(n p) (c_upper) and
 * ceil(n (1 - p)) (c_lower); an entry is an outlier iff w >= c_upper or w <= c_lower (ties
 * included).  W_sparse = W o M, W_dense = W - W_sparse (exact).  GANQ* quantizes W_dense; its
 * objective is ganq_objective(W_dense, Q, T, H) since W - (W~_dense + W_sparse) = W_dense - W~_dense.
 *
 * ganq_outlier_split: W (m x n fp32) -> W_dense (m x n), per-row cutoffs c_lower / c_upper (m),
 * CSR row offsets (m + 1 int64) of W_sparse, and its nnz (HOST; synchronises the stream).
 * INVALID_ARG: m < 1, n < 2, r not in (0, 1), null pointers; UNSUPPORTED: n > 57344 (one row of
 * keys must fit in shared memory).
 * ganq_outlier_csr: fills col_idx (int32, ascending within a row) and values (fp32) of W_sparse
 * (nnz entries, as returned above).  Async.
 * ganq_sparse_gemm_add: Y (p x m fp32) += X W_sparse^T, X p x n fp16 -- the sparse path of the
 * deployed GANQ* layer next to ganq_lut_gemm.  Async.
 */
ganq_status_t ganq_outlier_split(const float* W, int64_t m, int64_t n, double r, float* W_dense, float* c_lower,
                                 float* c_upper, int64_t* row_offsets, int64_t* nnz, void* stream);
ganq_status_t ganq_outlier_csr(const float* W, int64_t m, int64_t n, const float* c_lower, const float* c_upper,
                               const int64_t* row_offsets, int32_t* col_idx, float* values, void* stream);
ganq_status_t ganq_sparse_gemm_add(const int64_t* row_offsets, const int32_t* col_idx, const float* values,
                                   int64_t m, int64_t n, const uint16_t* X, int64_t p, float* Y, void* stream);

/* ---------------------------------------------------------------- NEXT-4: k-means T^0
 * ganq_kmeans_codebook: T (DEVICE fp32 m x 2^N, written) = per-row 1-D Lloyd k-means of W (DEVICE
 * fp32 m x n row-major) started from the fp32 min-max grid (R-6): `iters` iterations of
 * {nearest level, first index on ties; each non-empty level <- fp64 mean of its weights, rounded
 * to fp32; empty levels keep their value} (reading R-24 -- Algorithm 1 takes T^0 as an
 * input; k-means is the Euclidean-distance baseline of
 * the related work).  iters = 0
 * gives the grid itself.  Pass the result as ganq_opts_t.T0.  n_bits in [1, 4] (else
 * GANQ_ERR_UNSUPPORTED), iters >= 0.  Async on `stream`.
 */
ganq_status_t ganq_kmeans_codebook(const float* W, int64_t m, int64_t n, int n_bits, int iters, float* T,
                                   void* stream);

const char* ganq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GANQ_H_ */
